# pair-kernel A/B (run under gpurun): exp/libgrape_walk_<v>.so on bench --skipgram
set -u
mkdir -p gpurun_out
for c in 2 5; do
for v in "$@"; do
  GRAPE_WALK_LIB=$PWD/exp/libgrape_walk_$v.so timeout 900 python bench.py --config $c --skipgram 2000000 --steps 5 --warmup 3 --no-e2e --no-cpu --no-probe > gpurun_out/absg_${c}_$v.json 2> gpurun_out/absg_${c}_$v.err
  python - "$c" "$v" <<'PY'
import json, sys
c, v = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/absg_{c}_{v}.json").read().strip().splitlines()[-1])
    print(f"cfg{c} {v:8s} value {d['value']:.4g}  step {d['ms_per_step']:.2f} ms  pair kernel {d['pair_kernel']['ms']:.2f} ms")
except Exception as e:
    print(c, v, "FAILED", e, open(f"gpurun_out/absg_{c}_{v}.err").read()[-400:])
PY
done
done
