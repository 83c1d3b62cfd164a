# Tensor-core block pass (pts_i8w_kernel) vs the FP64 DMMA pass at C4 and C3, the
# tensor-block tests, and one ncu --set full capture of the tensor-core kernel.
for cfg in C4 C3; do
  timeout 300 python tools/profile_i8.py i8 $cfg 2>&1 | tail -1 | sed 's/^/i8   /'
  timeout 300 python tools/profile_i8.py fp64 $cfg 2>&1 | tail -1 | sed 's/^/fp64 /'
done
timeout 900 python -m pytest tests/test_gpu_tensor_block.py -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:pts_i8w_kernel' -s 1 -c 1 -o gpurun_out/ncu_i8w_r02 python tools/profile_i8.py > gpurun_out/ncu_i8w_r02.log 2>&1
echo "ncu rc=$?"
