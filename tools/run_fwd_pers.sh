# persistent forward (pf) vs the non-persistent forward (w1): parity vs the one-tile experiment + same-box timing
export TESS_FWD_ONLY=1
for a in "1 512 4 128 3" "2 1000 4 64 3" "1 136 3 128 3" "3 520 24 128 3" "4 392 40 64 3" "2 128 8 128 3" "3 256 50 64 3" "4 2048 96 128 3" "1 128 1 128 3" "1 8 2 64 3"; do
  timeout 30 tools/libvar/attn_check_pf $a | grep -E "fwd1 vs|FAIL|rror"; done
for r in 1 2 3; do for v in w1 pf; do echo "== $v"; timeout 60 tools/libvar/attn_check_$v 4 2048 96 128 20 | grep -E "two-tile"; done; done
