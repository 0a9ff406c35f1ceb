# forward softmax in two 64-key halves (TESS_ATTN_FWD_SPLIT): parity vs the one-tile experiment + same-box timing; phase trace of the unsplit kernel
export TESS_FWD_ONLY=1
for a in "1 512 4 128 3" "2 1000 4 64 3" "1 136 3 128 3" "3 520 24 128 3" "4 392 40 64 3" "2 128 8 128 3" "3 256 50 64 3" "4 2048 96 128 3"; do
  timeout 120 tools/libvar/attn_check_s1 $a | grep -E "fwd1 vs|FAIL|rror"; done
for r in 1 2; do for v in s0 s1 s1p1; do echo "== $v"; timeout 300 tools/libvar/attn_check_$v 4 2048 96 128 20 | grep -E "two-tile"; done; done
TESS_FWD_TRACE=1 timeout 120 tools/libvar/attn_check_ftr 4 2048 96 128 2 | grep -v "ms/iter"
