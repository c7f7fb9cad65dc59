OUT=gpurun_out/r2rows2; mkdir -p $OUT
for r in 86 96 103; do
  timeout 300 python bench.py --workload s512 --extras none --rows $r --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/b_$r.json 2>> $OUT/err
  python -c "import json; d=json.load(open('$OUT/b_$r.json')); print('s512 rows=$r', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" >> $OUT/summary.txt
done
for r in 0 64 128; do
  timeout 300 python bench.py --workload l256 --dtype f64 --extras none --rows $r --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/l_$r.json 2>> $OUT/err
  python -c "import json; d=json.load(open('$OUT/l_$r.json')); print('l256 f64 rows=$r', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" >> $OUT/summary.txt
done
cat $OUT/summary.txt
