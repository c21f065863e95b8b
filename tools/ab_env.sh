#!/bin/bash
# Bench sweep over one environment knob of the current build (twice each, interleaved), plus the
# 100-iteration pegase iterate of each value compared bitwise with the default's.
# usage (under gpurun): bash tools/ab_env.sh VAR v1 v2 ...   ("" = unset)
set -u
VAR=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
mkdir -p /tmp/ab
python tools/ab_state.py /tmp/ab/default.npz pegase2869 100 > /dev/null
for rep in 1 2; do
  for v in "$@"; do
    if [ -z "$v" ]; then unset $VAR; else export $VAR=$v; fi
    echo "== $VAR=$v"; SKIP_TESTS=1 bash tools/quick_bench.sh
    if [ $rep = 1 ]; then
      python tools/ab_state.py /tmp/ab/v.npz pegase2869 100 > /dev/null
      python -c "
import numpy as np
a, b = np.load('/tmp/ab/default.npz'), np.load('/tmp/ab/v.npz')
bad = [k for k in a.files if a[k].tobytes() != b[k].tobytes()]
print('   iterate vs default:', 'bitwise equal' if not bad else 'DIFFER in %s (max abs %s)' % (bad, max(float(np.max(np.abs(a[k] - b[k]))) for k in bad)))"
    fi
  done
done
