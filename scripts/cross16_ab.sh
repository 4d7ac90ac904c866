# fp16 mode A/B: current library vs a variant (FQ_LIB), alternating runs.
python -m pytest tests/test_gpu_attention.py -m gpu -q > gpurun_out/pt_c16.txt 2>&1
for r in 1 2 3; do
for x in "" build/variants/oldcross.so; do
  FQ_LIB=$x python bench.py --precision fp16 --no-cpu-baseline --no-micro --steps 8 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('lib=$x', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])" >> gpurun_out/cross16_ab.txt
done; done
