#!/bin/bash
# scripts/build_variant.sh NAME SRC "EXTRA nvcc flags": rebuild liblpbp.so with the flags applied to
# csrc/SRC (e.g. kernels.cu) into exp_libs/NAME.so, then restore the default build.
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2; FLAGS=$3
touch paper_1608_03589_b200/csrc/$SRC
make -s EXTRA="$FLAGS" > /dev/null
cp paper_1608_03589_b200/liblpbp.so exp_libs/$NAME.so
touch paper_1608_03589_b200/csrc/$SRC
make -s > /dev/null
