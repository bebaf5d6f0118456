#!/usr/bin/env bash
# Regenerates the golden fixtures under tests/golden/ from the UNMODIFIED
# reference (compiled in place by oracle/Makefile into oracle/_ref/).
# Requires /root/reference (this container only).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
repo="$(cd "$here/../.." && pwd)"
make -C "$repo/oracle" ref
for d in rng pack gate feedback update_clause epoch_par_w1 epoch_seq inference regression models; do
  rm -rf "$here/$d"
done
"$repo/oracle/_ref/ref_driver" golden "$here"
# Transcript of the same-source drop-in driver built against the reference.
"$repo/oracle/_ref/api_driver_ref" > "$here/api_driver_ref.txt"
# Transcripts of the host-companion driver (data_io, metrics, bench).
tmp="$(mktemp -d)"
"$repo/oracle/_ref/data_driver_ref" host "$tmp" > "$here/data_driver_host_ref.txt" 2>/dev/null
"$repo/oracle/_ref/data_driver_ref" bench > "$here/data_driver_bench_ref.txt" 2>/dev/null
rm -rf "$tmp"
# Transcript of the scripted `tm` command-line session (tests/cli_session.py)
# with our CLI source linked against the reference library.
(cd "$repo" && python -m tests.cli_session oracle/_ref/tm_ref all > "$here/cli_session_ref.txt")
