#!/bin/bash
# Builds the current sources with extra nvcc flags into build/NAME.so (A/B
# timing with scripts/gpu_ab.sh NAME=build/NAME.so).  usage: build_variant.sh NAME "FLAGS"
set -e
NAME=$1; FLAGS=$2
R=/tmp/var_$NAME
rm -rf $R; mkdir -p $R/pkg
cp -r $(dirname $0)/../include $R/
cp -r $(dirname $0)/../paper_2006_02602_b200/csrc $R/pkg/
rm -rf $R/pkg/lib
make -s -j8 -C $R/pkg/csrc EXTRA="$FLAGS" 2>&1 | grep -v "spill\|^$" || true
mkdir -p $(dirname $0)/../build
cp $R/pkg/lib/libcavity_b200.so $(dirname $0)/../build/$NAME.so
echo "built build/$NAME.so"
