#!/bin/bash
# One GPU round trip while iterating: GPU parity tests, then device-only bench lines.
# usage (via gpurun): bash tools/gpu_check.sh TAG [workloads...]
tag=${1:-chk}; shift
wls=${@:-c3}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
for w in $wls; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
tail -2 gpurun_out/${tag}_tests.log
for w in $wls; do python - "$w" "gpurun_out/${tag}_bench_$w.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['value'],1), d['unit'], 'stages', {k:round(v,4) for k,v in d['config'].get('stage_ms',{}).items()}, 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None)
except Exception as e: print(sys.argv[1], 'bench failed', e)
PY
done
