for v in ${VARIANTS:-base none none_now none_noact none_notma base_now}; do LORS_B200_LIB=$PWD/paper_2501_08582_b200/_native/exp/$v/liblors_b200.so timeout 300 python tools/exp_k1.py; done
