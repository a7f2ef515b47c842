E=$PWD/paper_2501_08582_b200/_native/exp
for args in "8192 11008 4096 64 sp24" "8192 11008 4096 64"; do
echo "== $args"; LORS_B200_LIB=$E/trace/liblors_b200.so timeout 300 python tools/trace_k1.py $args 2>&1 | grep -E "issuer iteration|transform period|xf |main completion|issuer wready|CTA0 warp"
done
