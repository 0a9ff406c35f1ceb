timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_epilogue.py -q -m gpu 2>&1 | tail -2
bash tools/run_ab.sh
