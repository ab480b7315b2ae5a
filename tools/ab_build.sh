#!/bin/bash
# Build the library of git revision $1 into ab/$2.so (A/B runs via BRMQ_LIB).
set -e
rev=$1; name=$2; root=$(git rev-parse --show-toplevel)
tmp=$(mktemp -d); git -C "$root" worktree add -q --detach "$tmp" "$rev"
(cd "$tmp" && python -c "from paper_1706_06940_b200.build import build_lib; build_lib()")
mkdir -p "$root/ab"; cp "$tmp/paper_1706_06940_b200/libbrmq.so" "$root/ab/$name.so"
git -C "$root" worktree remove --force "$tmp"
