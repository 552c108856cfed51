B="python bench.py --steps 1 --warmup 1 --no-agg --no-cpu-baseline --no-c4"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_fwd$|k_wgrad|k_bwd_conv|k_lz_bwd|k_lz_gram|k_lz_fwd$|k_head" --launch-skip 14 --launch-count 8 -o gpurun_out/r1_head2 $B > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out/*.ncu-rep
