#!/bin/bash
# Build the current csrc tree as a named variant library: bash tools/variant.sh NAME
set -e
name=$1
mkdir -p _variants
make -s -j8 -C paper_2505_13215_b200/csrc OUT=$PWD/_variants/lib_$name.so BUILD=$PWD/_variants/build_$name 2>&1 | grep -E "error" || true
ls -la _variants/lib_$name.so
