for T in ${TARGETS:-2048 2600 3000 3400}; do
  for P in c2 c4; do
    echo "== target=$T problem=$P"
    AGGMG_STREAM_TARGET=$T timeout 200 python tools/kernel_bench.py --problem $P --reps 10 --kinds 0,3 | python -c "
import json,sys; d=json.load(sys.stdin)
print(' '.join(f'{k}={v[\"frac_of_peak\"]:.3f}' for k,v in d.items()))"
  done
done
