B="python bench.py --steps 1 --warmup 1 --no-agg --no-cpu-baseline --no-c4"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_fwd$|k_wgrad|k_bwd_conv|k_lz_bwd|k_lz_gram|k_lz_fwd$|k_head|k_lz_mat" --launch-skip 14 --launch-count 9 -o gpurun_out/r1_full_b $B > gpurun_out/ncu5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rn_conv|k_rn_gn" --launch-skip 40 --launch-count 6 -o gpurun_out/r1_resnet python tools/c4_bench.py > gpurun_out/ncu6.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"fold_group_vec|move_rows" --launch-count 4 -o gpurun_out/r1_hbm python tools/state_bench.py > gpurun_out/ncu7.log 2>&1
ls -la gpurun_out/*.ncu-rep
