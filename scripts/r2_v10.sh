OUT=gpurun_out/r2v10; mkdir -p $OUT
timeout 240 python -m pytest tests/test_parity_gpu.py -q -x -k "3d_kernel_variants" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
RPL_VARIANT=2 timeout 240 python -m pytest tests/test_parity_gpu.py -q -x -k "domain_error_is_reported_3d or minimum_sizes_fp32" >> $OUT/pytest.log 2>&1; echo "dom rc=$?" >> $OUT/pytest.log
for v in 0 2; do for w in w384 l256; do
  RPL_VARIANT=$v timeout 120 python bench.py --workload $w --extras none --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_$v.json 2>> $OUT/err
  python -c "import json; d=json.load(open('$OUT/b_${w}_$v.json')); print('$w v$v', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> $OUT/summary.txt
done; done
cat $OUT/summary.txt; grep rc= $OUT/pytest.log
