for v in ${VARIANTS:-base np}; do echo "== $v"; LORS_B200_LIB=$PWD/paper_2501_08582_b200/_native/exp/$v/liblors_b200.so timeout 300 python tools/overhead_fit.py; done
