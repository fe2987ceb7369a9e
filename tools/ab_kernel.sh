# A/B of kernel variants through bench.py (value = 20 back-to-back launches on 1 GiB)
#   bash tools/ab_kernel.sh "R:kernel:ctas ..."
for i in 1 2; do
for cfg in $1; do IFS=: read R K C <<< "$cfg"
v=$(PAGECRYPT_KERNEL=$K PAGECRYPT_CTAS_PER_SM=$C timeout 120 python bench.py --no-extras --rounds $R --cpu-seconds 0.2 --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")
echo "R=$R kernel=$K ctas=$C -> $v"
done; done
