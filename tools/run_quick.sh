timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_attention.py -q -m gpu -k "layer or ln or block or headline or attention" 2>&1 | tail -3
