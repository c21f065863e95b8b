#!/bin/bash
# Materialise a kernel translation unit at a git revision for an A/B run (run HERE, before gpurun:
# .git does not travel to the GPU box; build/ is git-ignored but does).
# usage: bash tools/ab_from_rev.sh REV k_sweep.cu   ->  prints build/ab/REV-k_sweep.cu
set -eu
REV=$1; UNIT=$2
mkdir -p build/ab
OUT=build/ab/$(git rev-parse --short "$REV")-$UNIT
git show "$REV:paper_2310_13145_b200/csrc/$UNIT" > "$OUT"
echo "$OUT"
