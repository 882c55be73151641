#!/bin/bash
# build libgshare_b200.so of a git revision (or the working tree with 'wt') into variants/<name>.so
# usage: bash tools/build_variant.sh <rev|wt> <name> [extra nvcc flags]
set -e
REV=$1; NAME=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p $ROOT/variants
if [ "$REV" = "wt" ]; then SRC=$ROOT; else
  SRC=$(mktemp -d); git -C $ROOT archive $REV paper_2309_00558_b200/csrc include | tar -x -C $SRC; fi
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -I $SRC/include "$@" -shared -o $ROOT/variants/$NAME.so \
  $SRC/paper_2309_00558_b200/csrc/gs_kernel.cu $SRC/paper_2309_00558_b200/csrc/gs_host.cpp -lcudart
echo built variants/$NAME.so
