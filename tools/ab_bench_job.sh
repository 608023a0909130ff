#!/bin/bash
# A/B of prebuilt libdali.so variants (abso/libdali_<name>.so) on the headline
# bench: tools/ab_bench_job.sh "nameA nameB" [bench args]
set -u
NAMES=$1; shift
mkdir -p gpurun_out/abso
for rep in 1 2; do for v in $NAMES; do
  cp abso/libdali_$v.so paper_2602_03495_b200/libdali.so
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/abso/$v$rep.json 2> gpurun_out/abso/$v$rep.log
  python tools/bench_summary.py gpurun_out/abso/$v$rep.json "$v rep $rep"
done; done
