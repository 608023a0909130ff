#!/bin/bash
# A/B of an engine switch on the headline workload (run under gpurun):
#   tools/ab_job.sh VAR "valA valB" [extra bench args]
# Runs bench.py (3 timed steps, no CPU baseline) alternately A B A B with the
# environment variable VAR set to each value; prints value / e2e per run.
set -u
VAR=$1; VALS=$2; shift 2
O=gpurun_out/ab
mkdir -p $O
for rep in 1 2; do
  for v in $VALS; do
    env $VAR=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" \
      > $O/${VAR}_${v}_$rep.json 2> $O/${VAR}_${v}_$rep.log
    python - "$O/${VAR}_${v}_$rep.json" "$VAR=$v rep $rep" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "value", d["value"], "e2e", d["e2e"]["value"], "prefill", d.get("prefill_tokens_per_s"),
          "floor_frac", (d.get("offload_roofline") or {}).get("frac_of_floor"),
          "host", d.get("host_ms_per_step"), flush=True)
except Exception as ex:
    print(sys.argv[2], "FAILED", ex)
PY
  done
done
