# Full-model decode (bench.py full-model leg) under K3S planner knobs: default, no small-layer
# pairs, no CTA pairs, 64 KB staging cap.  Run under gpurun: bash scripts/full_pair_ab.sh
for cfg in ${CFGS:-"" "MQ_STACK_FORCE_PAIR_N=0" "MQ_STACK_PAIR=0" "MQ_STACK_XS_CAP_KB=64"}; do
  env $cfg timeout 400 python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu --no-hetero --no-prefill --no-quant --no-c1 --no-c2 > gpurun_out/fq.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/fq.json').read().strip().splitlines()[-1])
m=d['full_model_decode']['models']
print('$cfg', {k:{b:round(v['tok_s'],1) for b,v in m[k]['per_bits'].items()} for k in m})"
done
