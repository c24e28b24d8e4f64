#!/bin/bash
# launch list of the headline bench + ncu --set full of the headline step's kernels, summarised
# on the box (no bench line): bash tools/gpu_ncu_quick.sh <tag>
TAG=${1:-q}
mkdir -p gpurun_out/round2
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:"rk::|weights_kernel|split_kernel" -c 600 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-extra --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"row_fwd_split|col_split|row_inv_split|weights_kernel" -c 4 \
    -o gpurun_out/full_cfg5_$TAG -f python tools/profile_predict_cfg5.py 1 > /dev/null 2>&1
RK_EVIDENCE_OUT=gpurun_out/round2 python tools/summarize_round2.py $TAG > gpurun_out/round2/summarize_$TAG.log 2>&1
for k in col_split row_inv_split row_fwd_split weights_kernel; do
  python tools/ncu_regions.py gpurun_out/full_cfg5_$TAG.ncu-rep $k > gpurun_out/round2/regions_${k}_$TAG.txt 2>&1
done
python tools/ncu_lines.py gpurun_out/full_cfg5_$TAG.ncu-rep 60 > gpurun_out/round2/lines_cfg5_$TAG.txt 2>&1
rm -f gpurun_out/full_cfg5_$TAG.ncu-rep
