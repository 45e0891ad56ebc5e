for rep in 1 2 3; do for v in "$@"; do echo -n "lib$v: "; LSE_LIB_PATH=$PWD/paper_1409_7474_b200/_lib/liblse_b200$v.so bash tools/quick_bench.sh; done; done
