cd paper_2105_14500_b200/csrc/tools
timeout 120 ./attn_check 2 1000 4 64 3 | grep -E "CHECK|bitwise|dQ:|dK:|dV:"
timeout 300 ./attn_check 4 2048 96 128 10 | grep -E "ms/iter|CHECK"
timeout 300 ./attn_check 4 2048 96 128 10 | grep -E "ms/iter"
