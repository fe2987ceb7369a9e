# A/B of library builds on the descriptor-array probe: bash tools/ab_desc.sh "dirA dirB" "12,8" "0 2 3"
for i in 1 2; do for v in $1; do cp build/$v/libpagecrypt.so paper_2004_09252_b200/libpagecrypt.so
for c in ${3:-0}; do PAGECRYPT_CTAS_PER_SM=$c timeout 300 python tools/desc_probe.py ${2:-12} 2>&1 | sed "s/^/$v ctas=$c /"; done; done; done
