# exp2 share on the FMA pipe in the single-tile forward: same-box variants
export TESS_FWD_ONLY=1
for r in 1 2; do for v in 0 1 5 21; do echo "== p$v"; timeout 300 tools/libvar/attn_check_p$v 4 2048 96 128 20 | grep -E "fwd"; done; done
