# single-tile forward with overlapped unit transitions: parity (several shapes) + same-box timing
export TESS_FWD_ONLY=1
for a in "1 512 4 128 3" "2 1000 4 64 3" "1 136 3 128 3" "3 520 24 128 3" "4 392 40 64 3" "2 128 8 128 3" "3 256 50 64 3"; do
  timeout 120 tools/libvar/attn_check_x0 $a | grep -E "fwd1 vs|FAIL|rror"; done
for r in 1 2; do for v in p0 p1 x0 x1; do echo "== $v"; timeout 300 tools/libvar/attn_check_$v 4 2048 96 128 20 | grep -E "ms/iter"; done; done
