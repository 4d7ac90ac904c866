python -m pytest tests -m gpu -x -q -k "attention or c2 or parity or engine" > gpurun_out/pt31.txt 2>&1
for ns in 2 3; do
  FQ_XH_SELF_STAGES=$ns python bench.py --no-cpu-baseline --half none --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); f=d['roofline']['profile']['families']
print('self ns=$ns', round(d['value']), {k: round(v['us']) for k, v in f.items()})" >> gpurun_out/self_ab.txt
done
