# ncu launch list (gpu__time_duration + DRAM bytes) of one C2 bench round;
# summarise with tools/sweep_profile.py gpurun_out/${1:-ll}.csv
P="python tools/profile_round.py"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${1:-ll}.csv $P > gpurun_out/${1:-ll}.log 2>&1
