timeout 1200 python -m pytest tests/test_gpu_attention.py -q -m gpu 2>&1 | tail -3
