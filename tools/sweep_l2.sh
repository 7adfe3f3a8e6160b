#!/bin/bash
# Raster / L2-policy sweep of assoc_i8 on a C3 slice (timing only; run under gpurun).
#   SWEEP_CFGS="group:codes ..."  group 0 = default (pairs/2); codes -1 = default,
#   else panel | geno << 2 with 0 normal, 1 evict_last, 2 evict_first.
cd "${GRAFT_REPO_ROOT:-.}"
for cfg in ${SWEEP_CFGS:-0:-1 0:4 0:0 0:1 32:1 74:4 18:4 0:5 0:8}; do
  g=${cfg%%:*}
  c=${cfg##*:}
  if [ "$g" != "0" ]; then export PG_GROUP_C=$g; else unset PG_GROUP_C; fi  # <0: panel-stationary
  if [ "$c" != "-1" ]; then export PG_L2_CODES=$c; else unset PG_L2_CODES; fi
  echo "== group=$g codes=$c"
  if [ "${SWEEP_TOOL:-bench}" = "c5" ]; then
    timeout 300 python tools/bench_workloads.py --workload c5 --markers ${SWEEP_MARKERS:-262144} --steps 3 2>&1 \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
  else
    timeout 300 python bench.py --total-markers ${SWEEP_MARKERS:-524288} --steps ${SWEEP_STEPS:-4} --warmup 3 --no-e2e \
      --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], d['ms_per_step'], r['achieved'], d['clocks'])"
  fi
done
