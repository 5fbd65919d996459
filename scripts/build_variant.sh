#!/bin/bash
# Build a variant of lib/libucfvb.so with extra nvcc flags into scratch/ab/<name>.so (A/B timing):
#   bash scripts/build_variant.sh <name> -DMACRO=VALUE ...
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=/tmp/bv_$name
rm -rf $W; mkdir -p $W/pkg $W/include
cp -r $ROOT/paper_2510_25906_b200/csrc $ROOT/paper_2510_25906_b200/Makefile $W/pkg/
cp $ROOT/include/*.h $W/include/
sed -i "s|^NVFLAGS := -O3|NVFLAGS := $* -O3|" $W/pkg/Makefile
make -C $W/pkg -j8 > $W/build.log 2>&1 || { tail -20 $W/build.log; exit 1; }
mkdir -p $ROOT/scratch/ab
cp $W/pkg/lib/libucfvb.so $ROOT/scratch/ab/$name.so
grep -A1 "troubled_cellsILi9ELi2ELi3" $W/pkg/build/ptxas_solver.log | grep Used || true
