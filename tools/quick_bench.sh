#!/bin/bash
# build, GPU parity tests, and two bench lines (20 and 100 steps) summarised on one line each
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || { echo build failed; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  UCAC_REQUIRE_GPU=1 timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E .*Error|FAILED|passed|failed" | head -8
fi
for s in ${STEPS:-20 100}; do
  python bench.py --steps $s --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['steps'], 'ms/step %.4f' % d['ms_per_step'], 'it/s %.0f' % d['value'], 'e2e %.0f' % d['e2e']['value'],
      {k: round(v * 1e3, 1) for k, v in d['kernel_ms_per_step'].items()})"
done
