# backward passes: epilogue TMEM loads batched, accumulators released before the global stores (q4) vs q3: parity + harness timing + bench-step A/B
for a in "1 512 4 128 3" "2 1000 4 64 3" "1 136 3 128 3" "3 520 24 128 3" "4 392 40 64 3" "2 128 8 128 3" "1 256 50 64 3"; do
  echo "== q4 $a"; timeout 40 tools/libvar/attn_check_q4 $a | grep -E "kv\+dQpass|FAIL|rror"; done
for r in 1 2 3; do for v in q3 q4; do echo "== $v"; timeout 60 tools/libvar/attn_check_$v 4 2048 96 128 10 | grep -E "dQ pass|dK/dV pass  "; done; done
bash tools/run_ab.sh
