#!/usr/bin/env bash
# Build an A/B variant of the library with extra compile definitions, e.g.
#   tools/build_variant.sh direct0 -DRHG_SLAB_DIRECT=0
# -> build/variants/direct0/librhg_b200.so ; run with RHG_LIB_PATH=build/variants/direct0/librhg_b200.so
set -eu
NAME=$1; shift
OUT=build/variants/$NAME
mkdir -p "$OUT"
make -s -C paper_1710_07565_b200/csrc OUT="$PWD/$OUT/librhg_b200.so" OBJDIR="$PWD/$OUT/obj" EXTRA="$*" > "$OUT/build.log" 2>&1
echo "$OUT/librhg_b200.so"
