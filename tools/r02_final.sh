#!/bin/bash
# Final round-2 measurement on one B200 (run under gpurun): build, every GPU test, smoke, ncu --set
# full captures of every iteration kernel (pegase T=48; their DRAM bytes -> profiles/r02/
# ncu_traffic.json, which the bench line's roofline.traffic reads), the bench line, the reference
# arm, the ncu launch list of the bench command, the graph timeline, and the sweep kernels at
# T=168 (L2-free working set) for the HBM figures.
set -u
OUT=gpurun_out/${1:-final}; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo build failed; tail "$OUT/build.log"; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/smi.txt" 2>&1
UCAC_REQUIRE_GPU=1 timeout 1800 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest gpu rc=$?"; tail -3 "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"; tail -1 "$OUT/smoke.log"
for k in k_branch_al k_branch k_ubar k_rows k_bus k_genx k_bus_late k_rows_late k_fold_early; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^${k}(<|\$)" -s 4 -c 1 \
    -o "$OUT/full_$k" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttr-all > "$OUT/ncu_full_$k.log" 2>&1
  echo "ncu full $k rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_gen(<|\$)" -s 5 -c 1 \
  -o "$OUT/full_k_gen" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttr-all > "$OUT/ncu_full_k_gen.log" 2>&1
echo "ncu k_gen rc=$?"
python tools/ncu_traffic.py "$OUT" "ncu --set full --clock-control none, one launch each (the 5th of each kernel in bench.py --steps 2 --warmup 3: pegase T=48 graph iteration 5; k_gen: the 6th), tools/r02_final.sh" > "$OUT/ncu_traffic.json" && cp "$OUT/ncu_traffic.json" profiles/r02/ncu_traffic.json
timeout 900 python bench.py > "$OUT/bench.jsonl" 2> "$OUT/bench.err"; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > "$OUT/bench_reference.jsonl" 2> "$OUT/bench_reference.err"; echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttr-all > "$OUT/ncu_launches.log" 2>&1
echo "ncu launches rc=$?"
UCAC_EXTRA_NVCC="-DUCAC_PROF" python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
for r in 1 2 3; do python tools/timeline.py pegase2869 100 >> "$OUT/timeline.txt" 2>&1; done
python tools/al_timeline.py 100 > "$OUT/al_timeline.txt" 2>&1
python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
mkdir -p "$OUT/t168"
for k in k_rows k_bus k_ubar k_genx k_branch; do
  timeout 900 ncu --set full --clock-control none -k "regex:^${k}(<|\$)" -s 4 -c 1 \
    -o "$OUT/t168/full_$k" python bench.py --T 168 --steps 2 --warmup 3 --no-cpu-baseline --no-ttr-all > "$OUT/t168/ncu_$k.log" 2>&1
  echo "ncu t168 $k rc=$?"
done
timeout 900 python bench.py --T 168 --steps 20 --warmup 5 --no-cpu-baseline --no-ttr-all > "$OUT/bench_t168.jsonl" 2> "$OUT/bench_t168.err"; echo "bench t168 rc=$?"
