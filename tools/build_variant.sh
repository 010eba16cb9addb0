#!/bin/bash
# build the working tree with extra nvcc flags into ab/$1.so
set -e
name=$1; shift
root=/root/repo; tmp=$(mktemp -d); mkdir -p $root/ab
for f in $root/paper_2011_01112_b200/csrc/*.cu; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC "$@" -c "$f" -o "$tmp/$(basename "$f" .cu).o" &
done
wait
nvcc -shared -cudart static -gencode arch=compute_100a,code=sm_100a -o "$root/ab/$name.so" "$tmp"/*.o
rm -rf "$tmp"; echo built ab/$name.so
