SECS=3000 JOBS="C4:stable:8 C4:literal:8" CHUNK=2 bash tools/gpurun_oracle_bg.sh \
  'timeout 1500 python -m pytest tests -m gpu -q --durations=30 -p no:cacheprovider > gpurun_out/gputest3.log 2>&1' \
  'timeout 300 python tools/diag_stable_c3.py C3 > gpurun_out/diag_c3b.log 2>&1' \
  'timeout 600 python tools/tune_lse.py 4 5 19 20 21 24 40 41 42 43 44 45 46 47 201 204 206 210 211 212 214 215 > gpurun_out/tune3.log 2>&1' \
  'bash tools/gpurun_ncu.sh 3 pts_mma2_kernel 1 ncu_block_v2_r02'
