mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_stack.py tests/test_gpu_stack_parity.py -q -x > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pdl_tests.log
for v in 1 0; do
MQ_STACK_PDL=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-c2 --no-prefill --no-quant --no-cpu --no-hetero --no-c1 > gpurun_out/bench_full_pdl$v.json 2> gpurun_out/bench_full_pdl$v.err; echo "bench pdl=$v rc=$?"
python - <<PY
import json;d=json.loads(open("gpurun_out/bench_full_pdl$v.json").read().strip().splitlines()[-1]);f=d["full_model_decode"]
print("headline", round(d["value"],1), d["per_bits"]["4"]["stack_frac"])
for m,v in f["models"].items(): print(m, {k:round(x["tok_s"],1) for k,x in v["per_bits"].items()}, {k:(round(x,4) if isinstance(x,float) else x) for k,x in v["components_ms_r4"].items()})
PY
done
MQ_STACK_LAUNCH_DEBUG=1 timeout 300 python -c "
import torch
from paper_2602_03537_b200.llama import LlamaDecoder
from paper_2602_03537_b200.shapes import SHAPES
d=LlamaDecoder(batch=1, n_layers=2, vocab=1024)
d.capture(); d.step(); torch.cuda.synchronize(); print('ok')
" 2>&1 | tail -4
