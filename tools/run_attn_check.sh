cd paper_2105_14500_b200/csrc/tools
for r in 1 2; do
echo "== blocks"; timeout 300 ./attn_check 4 2048 96 128 10 | grep -E "dQ pass|dK/dV"
echo "== per-MMA"; timeout 300 ./attn_check_noblk 4 2048 96 128 10 | grep -E "dQ pass|dK/dV"
done
