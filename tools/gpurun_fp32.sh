set -x
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x 2>&1 | tail -15
timeout 600 python tools/fp32_probe.py 2>&1 | tail -12
