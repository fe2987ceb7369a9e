# Kernel-only durations (ncu launch list, cold, serialised) of the crypt kernel
# for kernel knobs and round counts: bash tools/ll_compare.sh "0 9" "20 12" [tag]
export PATH=/usr/local/cuda/bin:$PATH
for k in $1; do for r in $2; do
  PAGECRYPT_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 9 --csv \
    --log-file gpurun_out/ll_${3:-x}_k${k}_r${r}.csv python tools/profile_driver.py --rounds $r --launches 4 > /dev/null 2>&1
done; done
