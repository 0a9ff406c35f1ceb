# backward exp2 share on the FMA pipe (TESS_ATTN_BWD_POLY bit mask over every 4 exponentials; 8 = shipped, 1 in 4), same box
for r in 1 2 3; do for v in 0 8 10 12; do echo "== bp$v"; timeout 60 tools/libvar/attn_check_bp$v 4 2048 96 128 10 | grep -E "dQ pass|dK/dV pass  |kv\+dQpass dQ"; done; done
