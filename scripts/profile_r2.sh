#!/bin/bash
# Round-2 evidence capture on one B200 (run through gpurun): one ncu --set full of every
# k_decode (d-gap path) and k_index instantiation of configs 1-4 and the launch list of the
# default bench.  The reports are summarised on the box (raw metric CSV, traffic JSON, key
# metrics) and deleted, so gpurun_out/ stays small; the summaries go to profiles/.
set -u
mkdir -p gpurun_out/r2
rm -f profiles/r2_traffic.json.box
for c in ${CFGS:-1 2 3 4}; do
  case $c in 1) n=1;; 2) n=10;; 3) n=2;; 4) n=1;; esac
  timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --kernel-name 'regex:k_decode<.*, \(bool\)1, \(bool\)0>|k_index' --launch-count $((3 * n)) \
    -o /tmp/r2_cfg$c -f python bench.py --config $c --steps 1 --warmup 0 --no-e2e \
    --no-cpu-baseline --extra-configs none > gpurun_out/r2/ncu_cfg$c.log 2>&1
  echo "ncu cfg$c rc=$?"
  w=$(python -c "import gen; print(gen.config($c, scale=1e-4).name)")
  ncu -i /tmp/r2_cfg$c.ncu-rep --page raw --csv > gpurun_out/r2/raw_cfg$c.csv
  python scripts/ncu_summary.py full /tmp/r2_cfg$c.ncu-rep > gpurun_out/r2/full_cfg$c.md
  python scripts/ncu_summary.py traffic /tmp/r2_cfg$c.ncu-rep $w gpurun_out/r2/traffic.json
  python scripts/ncu_sass.py /tmp/r2_cfg$c.ncu-rep > gpurun_out/r2/sass_cfg$c.txt 2>/dev/null
  gzip -f gpurun_out/r2/raw_cfg$c.csv gpurun_out/r2/sass_cfg$c.txt
  rm -f /tmp/r2_cfg$c.ncu-rep
done
if [ -z "${CFGS:-}" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/r2/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e \
  --no-cpu-baseline --extra-configs none > gpurun_out/r2/launches.log 2>&1
echo "launches rc=$?"
fi
du -sh gpurun_out
