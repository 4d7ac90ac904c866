# GEMM A/B: current library vs build/variants/oldgemm.so (FQ_LIB), exact and
# fp16 benches alternating; full GPU tests first.
python -m pytest tests -m gpu -q -x > gpurun_out/pt_gemm.txt 2>&1
for r in 1 2 3; do
for x in "" build/variants/oldgemm.so; do
  FQ_LIB=$x python bench.py --no-cpu-baseline --no-micro --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('lib=$x', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], round(d['half_mode']['value']))" >> gpurun_out/gemm_ab.txt
done; done
