# A/B of library builds on the 1-page service latency sweep:
#   bash tools/ab_service.sh "S1 S4" [passes]
for i in $(seq 1 ${2:-2}); do for v in $1; do
  cp build/$v/libpagecrypt.so paper_2004_09252_b200/libpagecrypt.so
  timeout 300 python tools/service_workers_sweep.py 2000 2>/dev/null | sed "s/^/$v /"
done; done
