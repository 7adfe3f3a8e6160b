#!/bin/bash
# DRAM bytes per assoc_i8 launch for raster / L2 configs (ncu metrics pass; one gpurun call).
#   DRAM_CFGS="group:codes ..." as tools/sweep_l2.sh
cd "${GRAFT_REPO_ROOT:-.}"
CMD="python bench.py --total-markers 131072 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
for cfg in ${DRAM_CFGS:-74:5 -2:9}; do
  g=${cfg%%:*}
  c=${cfg##*:}
  export PG_GROUP_C=$g PG_L2_CODES=$c
  echo "== group=$g codes=$c"
  $CMD > /dev/null 2>&1 && ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:assoc_i8 -s 1 -c 1 $CMD 2>&1 | grep -E "dram__bytes_read|gpu__time|hit_rate"
done
