# ncu --set full (with source) of one dense-sweep launch of each conv kernel
# (sweep ~2 of the C2 bench round, ~830 active clients).
#   bash tools/ncu_conv.sh PREFIX
P="python tools/profile_round.py"
PFX=${1:-conv}
for k in k_bwd_conv k_wgrad k_fwd; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}\$" --launch-skip 2 --launch-count 1 -o gpurun_out/${PFX}_${k} $P > gpurun_out/${PFX}_${k}.log 2>&1
done
ls -la gpurun_out/${PFX}_*.ncu-rep
