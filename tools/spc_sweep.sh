CFGS=(${SPC_CFGS:-"148,74,37" "100,40,16" "120,50,20" "80,40,16" "200,74,37"})
for cfg in "${CFGS[@]}"; do
  PB_LZ_SPC=$cfg python bench.py --no-c4 --no-agg --no-cpu-baseline > gpurun_out/spc_$cfg.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/spc_$cfg.json')); k=d['kernels_ms_per_round']
print('$cfg', round(d['value'],3), round(d['ms_per_step'],2), 'lz_fwd', k['cnn_lz_fwd'], 'lz_bwd', k['cnn_lz_bwd'])"
done
