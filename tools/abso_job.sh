#!/bin/bash
# A/B of two prebuilt libdali.so variants (abso/libdali_<name>.so) on one box:
#   tools/abso_job.sh "nameA nameB" <command...>
set -u
NAMES=$1; shift
mkdir -p gpurun_out/abso
for rep in 1 2; do for v in $NAMES; do
  cp abso/libdali_$v.so paper_2602_03495_b200/libdali.so
  echo "== $v rep $rep"; "$@" 2>&1 | tail -6
done; done
