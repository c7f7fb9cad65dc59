#!/bin/bash
# ncu --set full captures (one launch each) of the dominant kernel of every row
TAG=${1:-ncurows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
# reports are summarised on the box (text only comes back: gpurun copies <= 64 MiB)
cap() { name=$1; regex=$2; shift 2; timeout 900 ncu --set full --clock-control none --import-source on -k regex:$regex -s 2 -c 1 -o $OUT/$name python bench.py --no-cpu-baseline --e2e-steps 0 --warmup 3 "$@" > $OUT/$name.log 2>&1;
  python tools/ncu_summary.py $OUT $name=$OUT/$name.ncu-rep > /dev/null 2>&1;
  python tools/sass_mix.py $OUT/$name.ncu-rep > $OUT/sass_mix_$name.txt 2>&1;
  rm -f $OUT/$name.ncu-rep; }
cap w384 k_step3d --workload w384 --steps 2
cap s512 k_step3d --workload s512 --steps 2
cap p6400 k_step2d_ra --workload p6400 --steps 2
cap o2_1024 k_step2d_o2 --workload o2_1024 --steps 3
cap o2_s256_xy k_step2d_o2 --workload o2_s256 --steps 2
cap o2_s256_z k_zmarch2 --workload o2_s256 --steps 2
cap fd8k_f64 k_fluxdiff_pt --workload fd8k --dtype f64 --steps 3
cap fd8k k_fluxdiff_ra --workload fd8k --steps 3
cap l256_f32_soa k_step3d --workload l256 --dtype f32 --steps 2
cap l256_f32_aos k_step3d --workload l256 --dtype f32 --layout aos --steps 2
cap l256_f64_soa k_step3d --workload l256 --dtype f64 --steps 2
cap l256_f64_aos k_step3d --workload l256 --dtype f64 --layout aos --steps 2
cap cfl1024 k_step2d_ra --workload cfl1024 --steps 2
ls -la $OUT; cat $OUT/ncu_*.txt
