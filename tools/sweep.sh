# C1..C5 device and end-to-end timings (one line per config)
for c in ${@:-C1 C2 C3 C4 C5}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['config']['workload'][:40], 'value', round(d['value'],3), 'ms/step', round(d['ms_per_step'],1), 'roof', round(r['frac'],3), 'share', round(r['kernel_share_of_step'],3), 'e2e', round(d['e2e']['value'],3), round(d['e2e']['partition_s'],3))
"
done
