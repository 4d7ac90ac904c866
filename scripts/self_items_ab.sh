# Exact-mode self-attention A/B: per-(item, head) kernel over shared history
# slots (FQ_XH_ITEMS_WARPS / _STAGES variants) vs the per-row kernel
# (FQ_SELF_ITEMS=0), alternating runs.
python -m pytest tests/test_gpu_attention.py -m gpu -q -k "items or self" > gpurun_out/pt_items.txt 2>&1
for w in 1 2; do FQ_XH_ITEMS_WARPS=$w python -m pytest tests/test_gpu_attention.py -m gpu -q -k "items" >> gpurun_out/pt_items.txt 2>&1; done
python -m pytest tests -m gpu -q -x -k "c2 or parity" >> gpurun_out/pt_items.txt 2>&1
for r in 1 2; do  # (defaults since: FQ_SELF_ITEMS=0, W=2, NS=3)
for x in "1 4 2" "1 2 2" "1 2 3" "0 4 2"; do set -- $x
  FQ_SELF_ITEMS=$1 FQ_XH_ITEMS_WARPS=$2 FQ_XH_ITEMS_STAGES=$3 python bench.py --half none --no-cpu-baseline --no-micro --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('items=$1 w=$2 ns=$3', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])" >> gpurun_out/self_items_ab.txt
done; done
FQ_SELF_ITEMS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:self_attention --csv --log-file gpurun_out/items_1.csv python bench.py --half none --no-cpu-baseline --no-micro --steps 1 --warmup 3 > /dev/null 2>&1
