#!/bin/bash
# ncu evidence for round 2 (run on the GPU box from the repo root, one GPU):
#   launch list of the N=1 headline bench, then one --set full capture of the headline
#   predict's kernels (K1 + 3 split-length passes, cfg5 4096^2 L=4 nu=2.5) and cfg3.
set -x
TAG=${1:-r2a}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"split_kernel|weights_kernel|row_fwd|col_kernel|row_inv" -c 12 \
    -o gpurun_out/full_cfg5_$TAG -f python tools/profile_predict_cfg5.py 2 > gpurun_out/ncu_full_cfg5_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/full_cfg5_$TAG.ncu-rep > gpurun_out/full_cfg5_${TAG}_summary.txt 2>&1
