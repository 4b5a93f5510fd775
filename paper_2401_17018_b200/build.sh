#!/usr/bin/env bash
# Builds libbdsm_b200.so in-tree for sm_100a (no torch types; plain C ABI).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
NVCC="${NVCC:-nvcc}"
FLAGS=(-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC
       -Xcompiler -fvisibility=hidden -I"$HERE/../include" --expt-relaxed-constexpr -diag-suppress 177
       ${BDSM_NVCC_EXTRA:-})
OBJ="${BDSM_OBJ:-$HERE/build}"
OUT="${BDSM_OUT:-$HERE/libbdsm_b200.so}"  # BDSM_OUT: alternative library (e.g. -DBDSM_TRACE diagnostics)
mkdir -p "$OBJ"
pids=()
for f in store match engine; do
  "$NVCC" "${FLAGS[@]}" -Xptxas -v -c "$HERE/csrc/$f.cu" -o "$OBJ/$f.o" 2> "$OBJ/$f.ptxas.log" &
  pids+=($!)
done
g++ -std=c++17 -O3 -fPIC -fvisibility=hidden -I"$HERE/../include" -I/usr/local/cuda/include \
    -c "$HERE/csrc/planner.cpp" -o "$OBJ/planner.o"
g++ -std=c++17 -O3 -fPIC -fvisibility=hidden -I"$HERE/../include" -c "$HERE/csrc/group.cpp" -o "$OBJ/group.o"
for p in "${pids[@]}"; do wait "$p" || { cat "$OBJ"/*.ptxas.log; exit 1; }; done
"$NVCC" -shared -gencode arch=compute_100a,code=sm_100a -o "$OUT" \
    "$OBJ/store.o" "$OBJ/match.o" "$OBJ/engine.o" "$OBJ/planner.o" "$OBJ/group.o" -lpthread
echo "built $OUT"
[ -n "${BDSM_OUT:-}" ] && exit 0
# `bdsm run` CLI (drop-in for the reference's tools/bdsm.cpp), linked against the C ABI
g++ -std=c++17 -O2 -I"$HERE/../include" "$HERE/csrc/cli.cpp" "$HERE/csrc/textio.cpp" \
    -L"$HERE" -lbdsm_b200 -Wl,-rpath,'$ORIGIN' -o "$HERE/bdsm"
echo "built $HERE/bdsm"
