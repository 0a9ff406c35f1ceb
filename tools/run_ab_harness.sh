# same-box comparison of attn_check builds in tools/libvar
for r in 1 2; do for v in A B; do echo "== $v"; timeout 300 tools/libvar/attn_check_$v 4 2048 96 128 10 | grep -E "attn_fwd|dQ pass|dK/dV pass  |PASS|FAIL|kv\+dQpass dQ"; done; done
timeout 120 tools/libvar/attn_check_B 2 1000 4 64 3 | grep -E "kv\+dQ"
