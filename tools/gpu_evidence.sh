#!/bin/bash
# Round-2 GPU evidence (run on the GPU box from the repo root, one GPU):
#   bench line (N=1), reference arm, ncu launch list of the bench, ncu --set full captures of the
#   headline predict (cfg5), cfg3, cfg2, K1 and the CS cfg4 ensemble kernels.
TAG=${1:-b}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:"rk::|weights_kernel|split_kernel" -c 600 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-extra --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"row_fwd_split|col_split|row_inv_split|weights_kernel" -c 4 \
    -o gpurun_out/full_cfg5_$TAG -f python tools/profile_predict_cfg5.py 1 > /dev/null 2>&1
for c in cfg3 cfg2; do
  ncu --set full --clock-control none --import-source on -k regex:"row_fwd|col_kernel<0|row_inv" --launch-skip 2 -c 3 \
      -o gpurun_out/full_${c}_$TAG -f python tools/profile_predict.py $c 3 > /dev/null 2>&1
  ncu --set full --clock-control none -k regex:"weights_kernel" -c 1 \
      -o gpurun_out/full_w_${c}_$TAG -f python tools/profile_weights.py $c 2 > /dev/null 2>&1
done
ncu --set full --clock-control none -k regex:"cs_|obs_local|accumulate|trmm|row_fwd|col_kernel|row_inv" -c 12 \
    -o gpurun_out/full_cs_$TAG -f python tools/cs_probe.py 64 32 > /dev/null 2>&1
# summarise on the box (ncu reports are too large to bring back), keep only the cfg5 capture
mkdir -p gpurun_out/round2
RK_EVIDENCE_OUT=gpurun_out/round2 python tools/summarize_round2.py $TAG > gpurun_out/round2/summarize.log 2>&1
python tools/ncu_regions.py gpurun_out/full_cfg5_$TAG.ncu-rep col_split > gpurun_out/round2/regions_col_split_$TAG.txt 2>&1
python tools/ncu_regions.py gpurun_out/full_cfg5_$TAG.ncu-rep row_inv_split > gpurun_out/round2/regions_row_inv_split_$TAG.txt 2>&1
python tools/ncu_regions.py gpurun_out/full_cfg5_$TAG.ncu-rep row_fwd_split > gpurun_out/round2/regions_row_fwd_split_$TAG.txt 2>&1
python tools/ncu_regions.py gpurun_out/full_cfg5_$TAG.ncu-rep weights_kernel > gpurun_out/round2/regions_weights_$TAG.txt 2>&1
rm -f gpurun_out/full_cfg3_$TAG.ncu-rep gpurun_out/full_cfg2_$TAG.ncu-rep gpurun_out/full_w_*_$TAG.ncu-rep gpurun_out/full_cs_$TAG.ncu-rep
du -sh gpurun_out/*
