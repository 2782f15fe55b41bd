#!/bin/bash
# Diagnostic: rebuild libgsgpc with different persistent-EFCG launch shapes and print the
# per-phase CG trace of configs 3, 5 and 2 (run on the GPU box: nvcc is in the image).
cd "$(dirname "$0")/.."
for v in "${@}"; do
  echo "=== variant: $v"
  python - <<PY
from paper_2101_11751_b200 import build as B
B.build(force=True, extra_flags="$v".split())
PY
  for c in 3 5 2; do
    GSGPC_CG_TRACE=1 python tools/profile_cg.py $c 300 2>&1 | grep -E "cg trace|ms/iter"
  done
done
python - <<PY
from paper_2101_11751_b200 import build as B
B.build(force=True)
PY
