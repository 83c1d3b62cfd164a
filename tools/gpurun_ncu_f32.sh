set -x
timeout 300 python tools/profile_lse.py 2 32 > gpurun_out/f32_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:pts_f32_kernel" -s 4 -c 1 -o gpurun_out/ncu_f32_r01 python tools/profile_lse.py 2 32 > gpurun_out/ncu_f32.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_f32.log
