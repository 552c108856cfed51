# Final-state evidence: full captures of the dense-sweep hot kernels, the
# launch list of one C2 round, and DRAM traffic per launch.
P="python tools/profile_round.py"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_fwd$|^k_bwd_conv$|^k_wgrad$|^k_lz_bwd|^k_lz_gram|^k_lz_fwd|^k_head$" --launch-skip 14 --launch-count 8 -o gpurun_out/final_dense $P > gpurun_out/final_dense.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $P > gpurun_out/final_launches.log 2>&1
ls -la gpurun_out/final_*
