#!/bin/bash
# A/B of an environment switch on one bench line (run under gpurun):
#   tools/ab_env_job.sh NAME "VAR=a VAR=b" [bench args]
# alternates the settings twice; prints tools/bench_summary.py per run.
set -u
NAME=$1; SETS=$2; shift 2
mkdir -p gpurun_out/abenv
for rep in 1 2; do for kv in $SETS; do
  env $kv timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" \
    > gpurun_out/abenv/${NAME}_${kv}_$rep.json 2> gpurun_out/abenv/${NAME}_${kv}_$rep.log
  python tools/bench_summary.py gpurun_out/abenv/${NAME}_${kv}_$rep.json "$NAME $kv rep $rep"
done; done
