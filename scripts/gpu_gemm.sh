set -x
timeout 600 python -m pytest tests/test_gpu_matmul.py -x -q 2>&1 | tail -25
timeout 600 python -m pytest tests/test_cpp.py -x -q -m gpu 2>&1 | tail -5
