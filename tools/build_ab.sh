#!/bin/bash
# Build libicsched.so from git revision $1 into ab/$2.so (A/B timing on one box:
# python bench.py --lib ab/$2.so ...).  Scratch tool; ab/ is git-ignored.
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2011_01112_b200/csrc include gen | tar -x -C "$tmp"
mkdir -p "$root/ab" "$tmp/obj"
for f in "$tmp"/paper_2011_01112_b200/csrc/*.cu; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -c "$f" -o "$tmp/obj/$(basename "$f" .cu).o" &
done
wait
nvcc -shared -cudart static -gencode arch=compute_100a,code=sm_100a -o "$root/ab/$name.so" "$tmp"/obj/*.o
rm -rf "$tmp"
echo "built ab/$name.so from $rev"
