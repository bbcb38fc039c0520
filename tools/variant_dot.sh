for v in $(ls build/variants); do echo "== $v"; AGGMG_LIB=build/variants/$v/libaggmg_b200.so timeout 100 python tools/dot_bench.py | grep chunked; done
