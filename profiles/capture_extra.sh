#!/bin/bash
# Run on the GPU box (gpurun): ncu evidence for the secondary rows under tag $1 (e.g. r02d):
# C3p (assign_labels + panoptic blend), the render backward, the C4 launch list.
tag=${1:-rXX}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python profiles/frame.py c3p 2 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"assign_labels|blend" --launch-skip 2 --launch-count 2 -o gpurun_out/x_c3p -f python profiles/frame.py c3p 2 > gpurun_out/x_c3p.log 2>&1
python profiles/summarize.py full gpurun_out/x_c3p.ncu-rep gpurun_out/${tag}_c3p_kernels_ncu.json
ncu --set full --import-source on --clock-control none -k regex:"backward|blend" --launch-skip 3 --launch-count 3 -o gpurun_out/x_bwd -f python tools/bench_backward.py c3 2 > gpurun_out/x_bwd.log 2>&1
python profiles/summarize.py full gpurun_out/x_bwd.ncu-rep gpurun_out/${tag}_backward_kernels_ncu.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x_c4.csv python profiles/frame.py c4 2 > /dev/null 2>&1
python profiles/summarize.py launches gpurun_out/x_c4.csv gpurun_out/${tag}_launches_c4_frame.csv
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x_c3p.csv python profiles/frame.py c3p 2 > /dev/null 2>&1
python profiles/summarize.py launches gpurun_out/x_c3p.csv gpurun_out/${tag}_launches_c3p_frame.csv
echo done
