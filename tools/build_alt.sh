#!/bin/bash
# build_alt.sh NAME "EXTRA nvcc/g++ flags": a library variant in build/alt/NAME.so for tools/gpu_ab.sh
set -e
cd "$(dirname "$0")/../paper_1710_07565_b200/csrc"
make -s -j8 OBJDIR=../../build/alt/$1 OUT=../../build/alt/$1.so EXTRA="$2" 2>&1 | grep -E "error" || true
ls -la ../../build/alt/$1.so
