for v in tile2 tile4 tile8; do
  for c in c2 c4; do
    AGGMG_LIB=build/variants/$v/libaggmg_b200.so timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu --no-prof | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', d['ms_per_step'], d['config']['setup_ms'], d['config']['solve_ms'])"
  done
done
