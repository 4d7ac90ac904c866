python -m pytest tests -m gpu -x -q -k "cross or c2 or parity" > gpurun_out/pt49.txt 2>&1
for ns in 3 4 6; do
  FQ_XH_CROSS_STAGES=$ns python bench.py --no-cpu-baseline --half none --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); f=d['roofline']['profile']['families']
print('ns=$ns', round(d['value']), {k: round(v['us']) for k, v in f.items()})" >> gpurun_out/cross_ab2.txt
done
