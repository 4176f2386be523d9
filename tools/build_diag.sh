#!/bin/bash
# Diagnostic builds of liblsgcpd.so (never the product): build/diag/lib_<name>.so with -D<flag>.
# Use with LSGCPD_LIB=build/diag/lib_<name>.so; results are wrong by construction.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/diag
for spec in "$@"; do
  name=${spec%%=*}; flag=${spec#*=}
  d=build/diag/$name; mkdir -p $d
  pids=()
  for f in paper_2103_15039_b200/csrc/*.cu; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
      --expt-relaxed-constexpr $(echo $flag | sed "s/,/ -D/g; s/^/-D/") -c $f -o $d/$(basename $f .cu).o &
    pids+=($!)
  done
  for p in "${pids[@]}"; do wait $p || { echo "compile failed for $name"; exit 1; }; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/diag/lib_$name.so $d/*.o -ldl
  rm -rf $d
done
