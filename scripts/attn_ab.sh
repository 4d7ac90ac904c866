# Attention A/B: current library vs build/variants/oldattn.so (FQ_LIB), exact
# bench alternating; attention + C2 tests first.
python -m pytest tests/test_gpu_attention.py tests/test_gpu_c2.py -m gpu -q > gpurun_out/pt_attn.txt 2>&1
for r in 1 2 3; do
for x in "" build/variants/oldattn.so; do
  FQ_LIB=$x python bench.py --half none --no-cpu-baseline --no-micro --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('lib=$x', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])" >> gpurun_out/attn_ab.txt
done; done
