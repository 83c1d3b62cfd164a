set -x
timeout 600 python -m pytest tests/test_gpu_api_surface.py -m gpu -q -x -k "sharded" 2>&1 | tail -5
timeout 900 python tools/c4_full_parity.py gpu 2>&1 | tail -5
ls -la gpurun_out/c4_full
