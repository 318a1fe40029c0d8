#!/usr/bin/env bash
# Builds libdiagsweep_b200.so for sm_100a (called by __graft_entry__.build()).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
out="${1:-$here/../lib/libdiagsweep_b200.so}"
mkdir -p "$(dirname "$out")"
NVCC="${NVCC:-nvcc}"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17
       -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr ${DS_EXTRA_FLAGS:-})
objs=()
tmp="$(mktemp -d)"
trap 'rm -rf "$tmp"' EXIT
for src in ds_assemble ds_core ds_factor ds_factor_blocked ds_modal ds_solve ds_stage ds_sweep; do
  "$NVCC" "${FLAGS[@]}" -DDS_BUILDING_LIB -c "$here/$src.cu" -o "$tmp/$src.o" &
  objs+=("$tmp/$src.o")
done
wait
CUDA_LIB="$(dirname "$(dirname "$(command -v "$NVCC")")")/lib64"
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared "${objs[@]}" -o "$out.tmp" -lcudart \
  -L"$CUDA_LIB" -Xlinker -rpath -Xlinker "$CUDA_LIB"
mv "$out.tmp" "$out"
echo "built $out"
