#!/bin/bash
# build a library variant: tools/build_variant.sh NAME "extra nvcc flags"
set -e
NAME=$1; shift
mkdir -p build_variants
rm -rf /tmp/gjv_$NAME && cp -r paper_1904_11201_b200 /tmp/gjv_$NAME && rm -rf /tmp/gjv_$NAME/build /tmp/gjv_$NAME/libgjoin.so
GJ_NVCC_EXTRA="$*" python -c "
import sys, native_build as nb
nb.PKG='/tmp/gjv_$NAME'; nb.CSRC=nb.PKG+'/csrc'; nb.LIB=nb.PKG+'/libgjoin.so'; nb.OBJDIR=nb.PKG+'/build'
nb.FLAGS=[f if f!=nb.CSRC else nb.CSRC for f in nb.FLAGS]
print(nb.build(force=True))"
cp /tmp/gjv_$NAME/libgjoin.so build_variants/libgjoin_$NAME.so
