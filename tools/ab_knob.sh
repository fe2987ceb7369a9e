# A/B of tuning knobs through the env (same build), alternating passes:
#   bash tools/ab_knob.sh "PAGECRYPT_KERNEL=0 PAGECRYPT_KERNEL=9,PAGECRYPT_CTAS_PER_SM=3" "20 12" [passes]
# (one config = comma-separated VAR=value list)
for i in $(seq 1 ${3:-2}); do for cfg in $1; do
  envs=$(echo $cfg | tr ',' ' ')
  for r in $2; do
    echo "$cfg R=$r bench $(env $envs timeout 120 python bench.py --no-extras --rounds $r --cpu-seconds 0.2 --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])")"
    env $envs timeout 120 python tools/desc_probe.py $r 2>/dev/null | sed "s/^/$cfg /"
  done
done; done
