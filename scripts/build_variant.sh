#!/bin/bash
# Build a variant of lib/libfkt_cuda.so with extra nvcc flags into
# lib_variants/<name>/ (developer A/B tool; load it with FKTB_LIB_PATH).
# usage: scripts/build_variant.sh <name> "<EXTRA_NVFLAGS>"
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=/tmp/fktb_variant_$NAME
rm -rf $TMP && mkdir -p $TMP
cp -r $ROOT/paper_2106_04487_b200/csrc $ROOT/paper_2106_04487_b200/cpp $ROOT/paper_2106_04487_b200/Makefile $TMP/
mkdir -p $TMP/../include && cp -r $ROOT/include/* $TMP/../include/ 2>/dev/null || true
make -s -j8 -C $TMP lib/libfkt_cuda.so EXTRA_NVFLAGS="$FLAGS" 2>&1 | grep -E " error" || true
mkdir -p $ROOT/lib_variants/$NAME
cp $TMP/lib/libfkt_cuda.so $ROOT/lib_variants/$NAME/
echo "built lib_variants/$NAME/libfkt_cuda.so"
