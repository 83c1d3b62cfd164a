set -x
timeout 300 python tools/profile_lse.py 0 32 cull > gpurun_out/cull32_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:pts_cull_kernel" -s 6 -c 1 -o gpurun_out/ncu_cull32_r01 python tools/profile_lse.py 0 32 cull > gpurun_out/ncu_cull32.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_cull32.log
