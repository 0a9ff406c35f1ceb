# single-tile forward (attn_fwd1) vs two-tile forward: parity and timing
cd paper_2105_14500_b200/csrc/tools
export TESS_FWD_ONLY=1
timeout 120 ./attn_check 1 512 4 128 3
timeout 120 ./attn_check 2 1000 4 64 3
timeout 120 ./attn_check 1 136 3 128 3
timeout 120 ./attn_check 3 520 24 128 3
timeout 120 ./attn_check 4 392 40 64 3
timeout 300 ./attn_check 4 2048 96 128 20
