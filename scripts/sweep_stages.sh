mkdir -p gpurun_out; rm -f gpurun_out/stages.txt
for d in 8 6 5 4 3 2; do
  MQ_STACK_MAX_STAGES=$d timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-prefill --no-full --no-hetero --no-quant > gpurun_out/st_$d.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/st_$d.json').read().strip().splitlines()[-1])
print('D<=$d', {k:round(v['tok_s'],1) for k,v in d['per_bits'].items()})" >> gpurun_out/stages.txt
done
