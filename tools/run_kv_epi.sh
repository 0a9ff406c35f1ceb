# dK/dV pass epilogue: the group's dK (then dV) half loaded with all TMEM loads in flight and one wait (ke) vs one wait per 16 columns (bp8 = shipped), same box, 4 alternations
for a in "1 512 4 128 3" "2 1000 4 64 3" "3 520 24 128 3" "4 392 40 64 3"; do
  echo "== ke $a"; timeout 40 tools/libvar/attn_check_ke $a | grep -E "kv\+dQpass|FAIL|rror"; done
for r in 1 2 3 4; do for v in bp8 ke; do echo "== $v"; timeout 60 tools/libvar/attn_check_$v 4 2048 96 128 20 | grep -E "dK/dV pass  |dK/dV pass \+"; done; done
