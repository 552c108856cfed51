set -x
B="python bench.py --steps 1 --warmup 1 --no-agg --no-cpu-baseline --no-c4"
# head sweep (sweep 2 of round 0) and tail sweep (sweep ~60) of key kernels
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_bwd_conv|k_lz_bwd|k_lz_gram|k_fwd$|k_wgrad" --launch-skip 10 --launch-count 5 -o gpurun_out/r1_head $B > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_head" --launch-skip 60 --launch-count 1 -o gpurun_out/r1_tailhead $B > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_lz_mat" --launch-count 1 -o gpurun_out/r1_mat $B > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out/*.ncu-rep
