# Repeat the default bench N times (no extras) and print one summary line per run.
for i in $(seq 1 ${1:-5}); do
  timeout 200 python bench.py --no-extras --cpu-seconds 0.5 2>/dev/null | tail -1 | RUN=$i python -c "
import json, os, sys
d = json.loads(sys.stdin.read())
print(json.dumps({'run': int(os.environ['RUN']), 'value': d['value'], 'frac': d['roofline']['frac'], 'e2e': d['e2e']['value'],
                  'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons'], 'power_w_max': d['clocks']['power_w_max']}))"
done
