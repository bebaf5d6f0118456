#!/usr/bin/env bash
# Builds alternative libtmgpu.so variants (tuning experiments) into
# paper_2009_04861_b200/_lib/variants/<name>/libtmgpu.so.
set -e
cd "$(dirname "$0")/.."
csrc=paper_2009_04861_b200/csrc
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  out="paper_2009_04861_b200/_lib/variants/$name"
  mkdir -p "$out"
  make -s -C $csrc OUT="$(pwd)/$out" EXTRA="$flags" -j8 >/dev/null
  echo "built $name ($flags)"
done
