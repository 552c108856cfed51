B="python bench.py --steps 1 --warmup 1 --no-agg --no-cpu-baseline --no-c4"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_fwd$|k_wgrad|k_bwd_conv|k_lz_bwd|k_lz_gram|k_lz_fwd$|k_head|k_lz_fold" --launch-skip 14 --launch-count 9 -o gpurun_out/r1c_cnn $B > gpurun_out/ncu8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rn_conv_tma|k_rn_wgrad_tma|k_rn_conv|k_rn_gn" --launch-skip 60 --launch-count 8 -o gpurun_out/r1c_resnet python tools/c4_bench.py > gpurun_out/ncu9.log 2>&1
timeout 1000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c2.csv $B > gpurun_out/ncu10.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_r1c2.csv
