# ncu --set full captures of single tail-sweep launches (sweep 64 of 72 in
# the bench round: 1-3 active clients) of the latency-bound kernels.
set -x
P="python tools/profile_round.py"
for spec in "k_head:64:1" "k_wgrad:64:1" "k_lz_gram:127:2" "k_lz_fwd_epi:20:1" "k_lz_bwd:64:1" "k_bwd_conv:64:1" "k_fwd:64:1" "k_lz_fwd:64:1"; do
  IFS=: read k skip cnt <<< "$spec"
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}\$|^${k}<" --launch-skip $skip --launch-count $cnt -o gpurun_out/tail_${k} $P > gpurun_out/tail_${k}.log 2>&1
done
ls -la gpurun_out/tail_*.ncu-rep
