for r in 1 2; do
for x in "2 3" "3 3" "2 4"; do set -- $x
  FQ_XH_SELF_STAGES=$1 FQ_XH_CROSS_STAGES=$2 python bench.py --half none --no-cpu-baseline --no-micro --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('self=$1 cross=$2', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])" >> gpurun_out/ns_ab.txt
done; done
