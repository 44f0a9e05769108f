#!/bin/bash
# Run on the GPU box (gpurun): every bench line of BASELINE.md's results table for round tag $1,
# then the profiles/capture.sh ncu evidence for the same tag.
tag=${1:-rXX}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 600 python bench.py > gpurun_out/${tag}_default.json 2> gpurun_out/${tag}_default.err
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err
for wl in c1 c2 c3p c4 c5; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/${tag}_${wl}.json 2> gpurun_out/${tag}_${wl}.err
done
timeout 1200 bash profiles/capture.sh $tag > gpurun_out/${tag}_capture.log 2>&1
echo "capture rc=$?" >> gpurun_out/${tag}_capture.log
