# bench C2 under several sparse-sweep thresholds (PB_CNN_TAIL=head,wgrad)
CFGS=(${TAIL_CFGS:-"60,60" "120,60" "200,60" "60,100" "60,150" "120,120"})
for cfg in "${CFGS[@]}"; do
  PB_CNN_TAIL=$cfg python bench.py --no-c4 --no-agg --no-c13 --no-cpu-baseline > gpurun_out/tail_$cfg.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/tail_$cfg.json')); k=d['kernels_ms_per_round']
print('$cfg', round(d['value'],3), round(d['ms_per_step'],2), 'head', k['cnn_head'], 'wgrad', k['cnn_wgrad'])"
done
