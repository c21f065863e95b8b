#!/bin/bash
# Bench sweep over compile-time variants (UCAC_EXTRA_NVCC), twice each, interleaved, with the
# 100-iteration pegase iterate of each compared bitwise with the first variant's.
# usage (under gpurun): bash tools/ab_build.sh "" "-DFOO=1" ...
set -u
mkdir -p /tmp/ab
for rep in 1 2; do
  i=0
  for v in "$@"; do
    UCAC_EXTRA_NVCC="$v" python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" || exit 1
    echo "== [$v]"; SKIP_TESTS=1 bash tools/quick_bench.sh
    if [ $rep = 1 ]; then
      python tools/ab_state.py /tmp/ab/v$i.npz pegase2869 100 > /dev/null
      python -c "
import numpy as np
a, b = np.load('/tmp/ab/v0.npz'), np.load('/tmp/ab/v$i.npz')
bad = [k for k in a.files if a[k].tobytes() != b[k].tobytes()]
print('   iterate vs first:', 'bitwise equal' if not bad else 'DIFFER in %s' % bad)"
    fi
    i=$((i+1))
  done
done
python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)"
