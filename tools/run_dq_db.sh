# dQ pass with dP double-buffered in TMEM (Q / dO as shared-memory A operands; q2) and + dP load overlapped with the exponentials (q3): parity + same-box timing vs the shipped pass (q0)
for a in "1 512 4 128 3" "2 1000 4 64 3" "1 136 3 128 3" "3 520 24 128 3" "4 392 40 64 3" "2 128 8 128 3" "1 256 50 64 3"; do
  echo "== q3 $a"; timeout 40 tools/libvar/attn_check_q3 $a | grep -E "kv\+dQpass dQ|FAIL|rror|non-finite"; done
for r in 1 2 3; do for v in q0 q2 q3; do echo "== $v"; timeout 60 tools/libvar/attn_check_$v 4 2048 96 128 10 | grep -E "dQ pass|dK/dV pass  "; done; done
