# dK/dV pass: dP^T load issued before the P^T store drain (k1) vs shipped (k0): parity + same-box timing
for a in "1 512 4 128 3" "2 1000 4 64 3" "1 136 3 128 3" "3 520 24 128 3" "4 392 40 64 3" "2 128 8 128 3" "1 256 50 64 3"; do
  echo "== k1 $a"; timeout 40 tools/libvar/attn_check_k1 $a | grep -E "kv\+dQpass|FAIL|rror"; done
for r in 1 2 3; do for v in k0 k1; do echo "== $v"; timeout 60 tools/libvar/attn_check_$v 4 2048 96 128 10 | grep -E "dQ pass|dK/dV pass  "; done; done
