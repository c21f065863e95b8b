#!/bin/bash
# A/B of a kernel change on the GPU: B = the working tree, A = an earlier revision of one translation
# unit (UCAC_SRC_OVERRIDE), materialised here first with tools/ab_from_rev.sh REV UNIT.
# Bench lines (quick_bench.sh, SKIP_TESTS=1) and the 100-iteration pegase / case300 iterates of both,
# compared bitwise.  usage (under gpurun): bash tools/ab_sweep.sh build/ab/<rev>-k_sweep.cu [k_sweep.cu]
set -u
OUT=/tmp/ab; mkdir -p $OUT gpurun_out/ab
A=$1
UNIT=${2:-k_sweep.cu}
for side in B A B A; do
  if [ $side = A ]; then export UCAC_SRC_OVERRIDE=$UNIT=$A; else unset UCAC_SRC_OVERRIDE; fi
  python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" || exit 1
  echo "== $side"; SKIP_TESTS=1 bash tools/quick_bench.sh
  for c in pegase2869 case300; do python tools/ab_state.py $OUT/$side-$c.npz $c 100 > /dev/null || exit 1; done
done
unset UCAC_SRC_OVERRIDE
python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)"
python - <<'PY'
import numpy as np
for c in ("pegase2869", "case300"):
    a, b = np.load(f"/tmp/ab/A-{c}.npz"), np.load(f"/tmp/ab/B-{c}.npz")
    bad = [k for k in a.files if a[k].tobytes() != b[k].tobytes()]
    print(c, "bitwise equal" if not bad else f"DIFFER in {bad}")
PY
UCAC_REQUIRE_GPU=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
# graph timelines of both sides (-DUCAC_PROF builds; diagnostic only)
for side in B A; do
  if [ $side = A ]; then export UCAC_SRC_OVERRIDE=$UNIT=$A; else unset UCAC_SRC_OVERRIDE; fi
  UCAC_EXTRA_NVCC=-DUCAC_PROF python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" || exit 1
  echo "== timeline $side"; python tools/timeline.py pegase2869 100 2>&1 | tail -16
done
unset UCAC_SRC_OVERRIDE
python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)"
