for v in a b a b; do echo "== $v"; HPLMM_LIB=$PWD/paper_2509_19777_b200/libhplmm_$v.so timeout 200 python tools/run_config.py cfg3 2>&1 | grep "solve 1"; done
