# Round-2 evidence in one GPU call: launch list + DRAM bytes of one C2 round,
# ncu --set full of the dense conv kernels, of the low-rank kernels (dense
# sweep 1-2 and a tail sweep), and of the C5 fold.
set -x
P="python tools/profile_round.py"
bash tools/launch_list.sh r2_ll
for k in k_bwd_conv k_wgrad k_fwd k_head; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}\$" --launch-skip 2 --launch-count 1 -o gpurun_out/r2_${k} $P > gpurun_out/r2_${k}.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_lz_" --launch-skip 8 --launch-count 6 -o gpurun_out/r2_lz_dense $P > gpurun_out/r2_lz_dense.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_lz_|^k_head_tail|^k_fwd$|^k_bwd_conv$|^k_wgrad$" --launch-skip 560 --launch-count 10 -o gpurun_out/r2_tail $P > gpurun_out/r2_tail.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"fold_group" --launch-skip 2 --launch-count 1 -o gpurun_out/r2_c5_fold python tools/c5_fold.py > gpurun_out/r2_c5_fold.log 2>&1
ls -la gpurun_out/r2_*
