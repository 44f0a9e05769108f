#!/bin/bash
# A/B timing of library variants on the GPU box: bash tools/ab.sh WORKLOAD ROUNDS base scratch/libpsm_X.so ...
# ("base" = the in-tree libpsm.so). Prints the blend / total stage times and frames/s of each run.
wl=$1; rounds=$2; shift 2
mkdir -p gpurun_out
for r in $(seq 1 $rounds); do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib="$PWD/$v"; fi
    PSM_LIB_PATH=$lib timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['config']['stage_ms']
print('$v', round(d['value'],1), 'blend', round(s['blend'],4), 'total', round(s['total'],4), 'pre', round(s['preprocess'],4), 'emit', round(s['emit'],4), 'sort', round(s['tile_sort'],4), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None)"
  done
done
