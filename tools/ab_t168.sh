#!/bin/bash
# A/B of compile-time variants at T = 168 and T = 48 (pegase): bench ms/step, interleaved twice,
# plus a graph timeline at T = 168 of each (-DUCAC_PROF).  usage (under gpurun): bash tools/ab_t168.sh "" "-DFOO=1" ...
set -u
for rep in 1 2; do
  for v in "$@"; do
    UCAC_EXTRA_NVCC="$v" python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" > /dev/null || exit 1
    for T in 168 48; do
      s=$([ $T = 168 ] && echo 20 || echo 100)
      python bench.py --T $T --steps $s --warmup 5 --no-cpu-baseline --no-ttr-all 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$v] T=$T steps=$s ms/step %.4f' % d['ms_per_step'], 'e2e %.0f' % d['e2e']['value'])"
    done
  done
done
for v in "$@"; do
  UCAC_EXTRA_NVCC="-DUCAC_PROF $v" python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" > /dev/null
  echo "== timeline T=168 [$v]"; python tools/timeline.py pegase2869 100 168 2>&1 | tail -11
done
python -c "from paper_2310_13145_b200 import build as b; b.build(force=True)" > /dev/null
