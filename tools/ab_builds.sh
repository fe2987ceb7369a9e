# A/B of library builds (build/<name>/libpagecrypt.so), alternating passes:
#   bash tools/ab_builds.sh "A B" "20 12" [ctas_per_sm] [passes]
# per build and round count: bench.py --no-extras (1 GiB contiguous, 20 launches)
# and tools/desc_probe.py (per-page descriptor shapes).
for i in $(seq 1 ${4:-2}); do for v in $1; do
  cp build/$v/libpagecrypt.so paper_2004_09252_b200/libpagecrypt.so
  for r in $2; do
    echo "$v R=$r bench $(PAGECRYPT_CTAS_PER_SM=${3:-0} timeout 120 python bench.py --no-extras --rounds $r --cpu-seconds 0.2 --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])")"
    PAGECRYPT_CTAS_PER_SM=${3:-0} timeout 120 python tools/desc_probe.py $r 2>/dev/null | sed "s/^/$v /"
  done
done; done
