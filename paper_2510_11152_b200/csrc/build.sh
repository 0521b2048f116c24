#!/usr/bin/env bash
# Build libfasmg_b200.so for sm_100a (in-tree, so it travels with gpurun).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
OUT="${HERE}/../libfasmg_b200.so"
NVCC="${NVCC:-nvcc}"
FLAGS=(-std=c++17 -O3 -lineinfo -fmad=false
       -gencode arch=compute_100a,code=sm_100a
       -Xcompiler -fPIC -Xptxas -warn-spills
       --expt-relaxed-constexpr -I"${HERE}")
OBJS=()
mkdir -p "${HERE}/../build"
for src in fasmg_runtime fasmg_natural fasmg_engine; do
  obj="${HERE}/../build/${src}.o"
  stale=0
  [[ -f "$obj" ]] || stale=1
  for dep in "${HERE}/${src}.cu" "${HERE}"/*.cuh "${HERE}"/*.h "${HERE}/build.sh"; do
    [[ "$dep" -nt "$obj" ]] && stale=1
  done
  if [[ $stale == 1 ]]; then
    "$NVCC" "${FLAGS[@]}" -c "${HERE}/${src}.cu" -o "$obj" &
  fi
  OBJS+=("$obj")
done
for job in $(jobs -p); do wait "$job"; done
for o in "${OBJS[@]}"; do [[ -f "$o" ]] || { echo "missing $o" >&2; exit 1; }; done
"$NVCC" -shared -gencode arch=compute_100a,code=sm_100a -o "$OUT" "${OBJS[@]}"
echo "built $OUT"
