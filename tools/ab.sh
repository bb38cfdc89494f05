timeout 1200 python -m pytest tests/test_gpu_farfield.py tests/test_gpu_parity.py tests/test_gpu_rays.py -x -q 2>&1 | tail -3
