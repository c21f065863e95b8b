#!/bin/bash
# Bench lines (100 and 20 steps), the reference arm and the ncu launch list of the bench command on
# the committed code (the tail of tools/r02_final.sh, without the ncu --set full captures).
set -u
OUT=gpurun_out/${1:-bench}; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo build failed; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"; tail -1 "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench.jsonl" 2> "$OUT/bench.err"; echo "bench rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > "$OUT/bench20.jsonl" 2> "$OUT/bench20.err"; echo "bench20 rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > "$OUT/bench_reference.jsonl" 2> "$OUT/bench_reference.err"; echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttr-all > "$OUT/ncu_launches.log" 2>&1
echo "ncu launches rc=$?"
