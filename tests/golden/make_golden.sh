#!/usr/bin/env bash
# Regenerates tests/golden/*.json from the UNMODIFIED reference (needs
# /root/reference, i.e. run in the build container, not on the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REPO="$(cd "$HERE/../.." && pwd)"
REF="${REF:-/root/reference/proj}"
make -C "$REPO/oracle" ref
BIN="$(mktemp -d)/make_golden"
g++ -std=c++20 -O2 -DNDEBUG -pthread -I"$REF/include" -I"$REF/tests" \
    -o "$BIN" "$HERE/make_golden.cpp" "$REPO/oracle/_ref/libbdsm_ref.a"
"$BIN" "$HERE"
ls -la "$HERE"/*.json
