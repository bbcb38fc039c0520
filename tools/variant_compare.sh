#!/bin/bash
# usage: tools/build_variant.sh <name> -DFOO=1 ...; then VARIANTS="<name>" bash tools/variant_compare.sh on the GPU box
# kernel_bench every built variant in build/variants/ (c2 and c4 problems)
for v in ${VARIANTS:-$(ls build/variants)}; do
  for P in ${PROBLEMS:-c2 c4}; do
    echo "== $v $P"
    AGGMG_LIB=build/variants/$v/libaggmg_b200.so timeout 200 python tools/kernel_bench.py --problem $P --reps 10 --kinds ${KINDS:-0,3} | python -c "
import json,sys; d=json.load(sys.stdin)
print(' '.join(f'{k}={v[\"avg_us\"]:.1f}us/{v[\"frac_of_peak\"]:.3f}' for k,v in d.items()))"
  done
done
