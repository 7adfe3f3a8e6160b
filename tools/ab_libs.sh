#!/bin/bash
# A/B of two builds of the library on the same box: copies ab/lib$X.so over the in-tree
# library before each run (newer mtime: bench.py's build check keeps it) and prints the C3
# device rate, GEMM ms and SM clock. Usage (under gpurun): AB_ORDER="A B A B" bash tools/ab_libs.sh
cd "${GRAFT_REPO_ROOT:-.}"
for x in ${AB_ORDER:-A B A B}; do
  cp ab/lib$x.so paper_2604_21095_b200/_lib/libpanelgwas_b200.so
  timeout 300 python bench.py --steps ${AB_STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline ${AB_ARGS} > gpurun_out/ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$x', d['value'], d['gemm_ms_per_step'], d['clocks']['sm_mhz'], d['value'] / d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.log
done
