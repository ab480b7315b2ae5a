#!/bin/bash
# Build the working tree once per compile-flag variant into ab/<name>.so
# (A/B runs via BRMQ_LIB, e.g. tools/ab_contract.py).
#   tools/ab_variants.sh base "" mb3 "-DBRMQ_CONTRACT_MINB=3" ...
set -e
root=$(git rev-parse --show-toplevel); cd "$root"; mkdir -p ab
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  BRMQ_NVCC_EXTRA="$flags" python -c "from paper_1706_06940_b200.build import build_lib; build_lib(force=True)"
  cp paper_1706_06940_b200/libbrmq.so "ab/$name.so"
done
python -c "from paper_1706_06940_b200.build import build_lib; build_lib(force=True)"
