#!/usr/bin/env bash
# Compile the reference headers' inline functions (the only executable code the
# headers-only reference has) and record their outputs as golden vectors.
# Runs only where /root/reference exists; output is committed.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REF:-/root/reference/proj/core/include}"
OUT="$HERE/../_ref"
mkdir -p "$OUT"
g++ -std=c++20 -O1 -I"$REF" "$HERE/ref_inline_pins.cpp" -o "$OUT/ref_inline_pins"
"$OUT/ref_inline_pins" > "$HERE/../../tests/golden/ref_inline_pins.json"
echo "wrote tests/golden/ref_inline_pins.json"
