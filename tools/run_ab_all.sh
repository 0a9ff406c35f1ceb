cd paper_2105_14500_b200/csrc/tools
timeout 120 ./attn_check 2 1000 4 64 3 | grep -E "kv\+dQ"
timeout 120 ./attn_check 1 136 3 128 3 | grep -E "kv\+dQ"
timeout 300 ./attn_check 4 2048 96 128 10 | grep -E "kv\+dQpass|dQ pass|dK/dV"
cd ../../..
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_headline.py -q -m gpu 2>&1 | tail -2
bash tools/run_ab.sh
