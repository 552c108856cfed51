# ncu --set full captures of single tail-sweep launches (sweep ~64 of 72 in
# the bench round: 4-6 active clients) of the latency-bound kernels.
#   bash tools/ncu_tail.sh PREFIX
set -x
P="python tools/profile_round.py"
PFX=${1:-tail}
for spec in "k_head_tail:34:1" "k_wgrad:64:1" "k_lz_gram:127:2" "k_lz_fwd_epi:20:1" "k_lz_bwd:64:1" "k_bwd_conv:64:1" "k_fwd:64:1" "k_lz_fwd:64:1"; do
  IFS=: read k skip cnt <<< "$spec"
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}\$|^${k}<" --launch-skip $skip --launch-count $cnt -o gpurun_out/${PFX}_${k} $P > gpurun_out/${PFX}_${k}.log 2>&1
done
ls -la gpurun_out/${PFX}_*.ncu-rep
