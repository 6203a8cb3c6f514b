# configs[1] layout-vs-speed table on the current walker (run under gpurun)
set -u
mkdir -p gpurun_out
bash tools/layout_sweep.sh 2 auto \
  "record_bytes=32,guide_bytes=32,guide_factor=8" "record_bytes=32,guide_bytes=32,guide_factor=4" \
  "record_bytes=32,guide_bytes=32,guide_factor=2" "record_bytes=32,guide_bytes=32,guide_factor=1" \
  "record_bytes=32,guide_bytes=8,guide_factor=4" "record_bytes=32,guide_bytes=8,guide_factor=1" \
  "record_bytes=16,guide_bytes=8,guide_factor=4" "record_bytes=16,guide_bytes=8,guide_factor=1"
timeout 600 python bench.py --config 2 --no-cpu --no-e2e --steps 3 --no-tables > gpurun_out/ls_cfg2_notables.json 2> gpurun_out/ls_cfg2_notables.err
python tools/show.py gpurun_out/ls_cfg2_notables.json | sed "s|^|no-tables |" | cut -c1-200
