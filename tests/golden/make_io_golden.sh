#!/bin/bash
# Regenerates tests/golden/io_golden.tsv from the unmodified reference file
# formats (oracle/_ref/ref_io_golden, built by `make -C oracle ref_io` from
# /root/reference). Test infrastructure only; run in the build container.
set -e
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
make -C "$ROOT/oracle" ref_io >/dev/null
make -C "$ROOT/tests/cpp" build/test_io >/dev/null
OUT="$ROOT/tests/golden/io_golden.tsv"
"$ROOT/oracle/_ref/ref_io_golden" > "$OUT"
# cross-reading: the drop-in's dictionary writer, read by the reference
TMP="$(mktemp)"
"$ROOT/tests/cpp/build/test_io" emit-dict "$TMP"
python3 -c "import sys; print('crossread\twriter\t' + open(sys.argv[1], 'rb').read().hex())" "$TMP" >> "$OUT"
printf 'crossread\treference_reads\t%s\n' "$("$ROOT/oracle/_ref/ref_io_golden" read-dict "$TMP")" >> "$OUT"
rm -f "$TMP"
wc -l "$OUT"
