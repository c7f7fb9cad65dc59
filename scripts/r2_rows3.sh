OUT=gpurun_out/r2rows3; mkdir -p $OUT
run() { timeout 300 python bench.py --workload $1 $3 --extras none --rows $2 --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/b_$1_$2.json 2>> $OUT/err; python -c "import json; d=json.load(open('$OUT/b_$1_$2.json')); print('$1 $3 rows=$2', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" >> $OUT/summary.txt; }
for r in 0 34 40 48 52; do run l256 $r "--dtype f64"; done
for r in 0 41 43 45 36; do run w384 $r; done
for r in 0 32 40 48; do run l256 $r; done
cat $OUT/summary.txt
