timeout 1500 python -m pytest tests/test_cli.py tests/test_gpu_streaming.py -m gpu -x -q 2>&1 | tail -3
