# A/B of library builds through bench.py: bash tools/ab_so.sh "dirA dirB" "R1 R2" [ctas]
for i in 1 2; do for v in $1; do cp build/$v/libpagecrypt.so paper_2004_09252_b200/libpagecrypt.so
for r in $2; do echo "$v R=$r $(PAGECRYPT_CTAS_PER_SM=${3:-0} timeout 120 python bench.py --no-extras --rounds $r --cpu-seconds 0.2 --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])")"; done; done; done
