for v in ${SG_VARIANTS:-sg0 sg1 sg0 sg1}; do
  for c in 2 5; do
    GRAPE_WALK_LIB=$PWD/exp/libgrape_walk_$v.so python bench.py --config $c --skipgram 2000000 --steps 3 --warmup 3 --no-cpu > gpurun_out/sgab_${v}_$c.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/sgab_${v}_$c.json').read().strip().splitlines()[-1]); print('$v', $c, round(d['pair_kernel']['ms'],2), round(d['streamed']['ms'],2), round(d['roofline']['frac'],3))"
  done
done
