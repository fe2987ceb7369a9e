# One ncu --set full capture of each kernel the bench line reports (the
# second launch of tools/profile_driver.py, default kernel per round count),
# contiguous and with per-page descriptor arrays: bash tools/ncu_bench_kernels.sh
export PATH=/usr/local/cuda/bin:$PATH
for r in 20 12 8; do
  for d in "" "--desc"; do
    tag=c$r${d:+_desc}
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_crypt_pages -s 1 -c 1 \
      -o gpurun_out/ncu_$tag python tools/profile_driver.py --rounds $r --launches 3 $d > /dev/null 2>&1
  done
done
ls gpurun_out/ncu_c*.ncu-rep
