for i in 1 2; do for cfg in "A 0" "A 3" "LB4 0" "LB4 3" "LB4 4"; do set -- $cfg
cp build/$1/libpagecrypt.so paper_2004_09252_b200/libpagecrypt.so
PAGECRYPT_CTAS_PER_SM=$2 timeout 120 python tools/desc_probe.py 12 2>/dev/null | sed "s/^/$1 ctas=$2 /"
done; done
