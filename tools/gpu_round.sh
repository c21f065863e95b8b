#!/bin/bash
# One GPU measurement round (run under gpurun from the repo root):
# build, gpu tests, smoke, bench, launch list, one ncu --set full capture per named kernel.
# Usage: tools/gpu_round.sh TAG [kernel ...]
set -u
TAG=${1:-run}; shift || true
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo build failed; tail "$OUT/build.log"; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/smi.txt" 2>&1
if [ -z "${SKIP_TESTS:-}" ]; then
  UCAC_REQUIRE_GPU=1 timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest gpu rc=$?"; tail -3 "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
fi
timeout 600 python bench.py > "$OUT/bench.jsonl" 2> "$OUT/bench.err"; rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > "$OUT/bench_reference.jsonl" 2> "$OUT/bench_reference.err"
echo "reference rc=$?"; tail -c 600 "$OUT/bench_reference.jsonl"
echo "bench rc=$rc"; tail -c 3000 "$OUT/bench.jsonl"
[ $rc -eq 0 ] || { tail -20 "$OUT/bench.err"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
echo "ncu launches rc=$?"
for k in "$@"; do
  # kernel names match as a regex on the function name (k_branch is a template: k_branch<false>)
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^${k}(<|\$)" -s 3 -c 1 \
    -o "$OUT/full_$k" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_full_$k.log" 2>&1
  echo "ncu full $k rc=$?"
done
