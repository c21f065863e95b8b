#!/bin/bash
# Round-2 measurement pass (run under gpurun from the repo root): bench lines, the graph timeline
# of one iteration (-DUCAC_PROF build), the ncu launch list and --set full captures of the sweep
# kernels VERDICT r01 asked for (k_ubar, k_rows, k_gen) plus the dominant ones.
# usage: tools/r02_profile.sh TAG [kernel ...]
set -u
TAG=${1:-prof}; shift || true
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo build failed; tail "$OUT/build.log"; exit 1; }
SKIP_TESTS=1 STEPS="20 100" bash tools/quick_bench.sh > "$OUT/quick.txt" 2>&1; cat "$OUT/quick.txt"
UCAC_EXTRA_NVCC="-DUCAC_PROF" python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
python tools/timeline.py pegase2869 100 > "$OUT/timeline.txt" 2>&1; cat "$OUT/timeline.txt"
python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
if [ -n "${NCU_LIST:-}" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?"
fi
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^${k}(<|\$)" -s ${NCU_SKIP:-4} -c 1 \
    -o "$OUT/full_$k" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_full_$k.log" 2>&1
  echo "ncu full $k rc=$?"
done
