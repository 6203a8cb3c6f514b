# per-rank launch time of strong-scaling slices, emulated on one GPU (run under gpurun):
# every rank slice of N = 2, 4, 8 for configs[1] and configs[4]
set -u
mkdir -p gpurun_out
for c in 2 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-probe > gpurun_out/slice_c${c}_full.json 2> gpurun_out/slice_c${c}_full.err
  ns="2 4 8"; [ $c = 5 ] && ns="8"
  for n in $ns; do
    for r in $(seq 0 $((n-1))); do
      timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-probe --slice $r/$n > gpurun_out/slice_c${c}_${r}of${n}.json 2> gpurun_out/slice_c${c}_${r}of${n}.err
    done
  done
done
python - <<'PY'
import json, glob
for c in (2, 5):
    full = json.loads(open(f"gpurun_out/slice_c{c}_full.json").read().strip().splitlines()[-1])
    T1 = full["ms_per_step"]
    print(f"config {c}: N=1 {T1:.2f} ms/step")
    for n in ((2, 4, 8) if c == 2 else (8,)):
        ms = []
        for r in range(n):
            d = json.loads(open(f"gpurun_out/slice_c{c}_{r}of{n}.json").read().strip().splitlines()[-1])
            ms.append(d["ms_per_step"])
        print(f"  N={n}: rank ms {[round(x, 2) for x in ms]}  max {max(ms):.2f}  predicted efficiency T1/(N max) = {T1 / (n * max(ms)):.3f}")
PY
