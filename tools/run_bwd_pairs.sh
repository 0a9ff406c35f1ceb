# backward exp2 share on the FMA pipe as packed pairs (exp2_fma2; TESS_ATTN_BWD_PAIRS over every 4 pairs) vs the shipped scalar 1-in-4 (pp1), same box
for a in "1 512 4 128 3" "2 1000 4 64 3" "3 520 24 128 3" "4 392 40 64 3"; do
  echo "== pp10 $a"; timeout 40 tools/libvar/attn_check_pp10 $a | grep -E "kv\+dQpass dQ|non-finite -> |FAIL|rror"; done
for r in 1 2 3; do for v in pp1 pp8 pp10 pp5 pp14; do echo "== $v"; timeout 60 tools/libvar/attn_check_$v 4 2048 96 128 20 | grep -E "dQ pass|dK/dV pass  |dK/dV pass \+"; done; done
