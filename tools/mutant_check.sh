#!/bin/bash
# Mutation check of the parity suite: build liblamb.so with a deliberately
# wrong pass B (chunk_b in csrc/lamb_kernels.cu) and show that the GPU parity tests FAIL.
#   nowd : pass B recomputes u without the decoupled weight-decay term (lambda * w)
#   scale: pass B applies 1.005 x the update
# Each mutant is built in a scratch copy of the repo; the real tree is untouched.
# Usage (GPU box): bash tools/mutant_check.sh > gpurun_out/mutants.log 2>&1
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TESTS="tests/test_gpu_parity.py::test_toy_parity tests/test_gpu_parity.py::test_random_ragged_tables tests/test_gpu_parity.py::test_gpt13b_layout_1p3b_full_size_sampled"
for mut in nowd scale; do
  W=/tmp/lamb_mutant_$mut
  rm -rf "$W"; mkdir -p "$W"
  (cd "$ROOT" && tar --exclude=./gpurun_out --exclude=./.git -cf - .) | (cd "$W" && tar -xf -)
  F="$W/paper_2402_15627_b200/csrc/lamb_kernels.cu"
  if [ $mut = nowd ]; then
    python3 - "$F" <<'PY'
import sys
p = sys.argv[1]; s = open(p).read()
old = "for (int q = 0; q < 4; ++q) ww[q] = __fmaf_rn(-scale, lamb_update(mm[q], vv[q], ww[q], G), ww[q]);"
assert old in s
s = s.replace(old, "GroupConst G0 = G; G0.wd = 0.f;\n    for (int q = 0; q < 4; ++q) ww[q] = __fmaf_rn(-scale, lamb_update(mm[q], vv[q], ww[q], G0), ww[q]);")
open(p, "w").write(s)
PY
  else
    python3 - "$F" <<'PY'
import sys
p = sys.argv[1]; s = open(p).read()
old = "for (int q = 0; q < 4; ++q) ww[q] = __fmaf_rn(-scale, lamb_update(mm[q], vv[q], ww[q], G), ww[q]);"
assert old in s
s = s.replace(old, "for (int q = 0; q < 4; ++q) ww[q] = __fmaf_rn(-scale * 1.005f, lamb_update(mm[q], vv[q], ww[q], G), ww[q]);")
open(p, "w").write(s)
PY
  fi
  rm -f "$W/paper_2402_15627_b200/liblamb.so"
  (cd "$W" && python3 -m paper_2402_15627_b200.build --force > /dev/null) || { echo "MUTANT $mut: build failed"; continue; }
  echo "== MUTANT $mut"
  (cd "$W" && timeout 900 python3 -m pytest $TESTS -q -m gpu -p no:randomly 2>&1 | grep -E "passed|failed|Error|out of tolerance" | head -20)
done
