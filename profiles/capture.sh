#!/bin/bash
# Run on the GPU box (gpurun): the ncu evidence committed under profiles/ for round tag $1 (e.g. r01b).
#  1. launch list of the bench command itself (gpu__time_duration per launch, cold and serialised)
#  2. launch list of one device-resident C3 frame (profiles/frame.py)
#  3. --set full of every kernel of that frame (the last of 2 frames)
set -e
tag=${1:-rXX}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_bench_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_frame.csv \
    python profiles/frame.py c3 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -o gpurun_out/${tag}_frame_full -f \
    python profiles/frame.py c3 2 > gpurun_out/${tag}_full.log 2>&1
python profiles/summarize.py full gpurun_out/${tag}_frame_full.ncu-rep gpurun_out/${tag}_c3_kernels_ncu.json
python profiles/summarize.py launches gpurun_out/${tag}_launches_frame.csv gpurun_out/${tag}_launches_c3_frame.csv
python profiles/summarize.py launches gpurun_out/${tag}_launches_bench.csv gpurun_out/${tag}_launches_c3_bench.csv
# bench.py's roofline.traffic comes from this same capture
python profiles/summarize.py traffic gpurun_out/${tag}_c3_kernels_ncu.json profiles/blend_traffic.json
cp profiles/blend_traffic.json gpurun_out/${tag}_blend_traffic.json
echo captured
