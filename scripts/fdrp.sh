#!/bin/bash
TAG=${1:-fdrp}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "flux" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -n 2 $OUT/pytest.log
bash scripts/tune.sh $TAG/t fd8k:0 fd8k:20 fd8k:73 fd1k:0 fd1k:20 fd16k:20
cap() { name=$1; regex=$2; shift 2; timeout 900 ncu --set full --clock-control none --import-source on -k regex:$regex -s 2 -c 1 -o $OUT/$name python bench.py --no-cpu-baseline --e2e-steps 0 --warmup 3 "$@" > $OUT/$name.log 2>&1;
  python tools/ncu_summary.py $OUT $name=$OUT/$name.ncu-rep > /dev/null 2>&1;
  python tools/sass_mix.py $OUT/$name.ncu-rep > $OUT/sass_mix_$name.txt 2>&1; rm -f $OUT/$name.ncu-rep; }
cap fd8k_rp k_fluxdiff_rp --workload fd8k --steps 3
cat $OUT/ncu_fd8k_rp.txt; head -12 $OUT/sass_mix_fd8k_rp.txt
