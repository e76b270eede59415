#!/bin/bash
# Builds a variant of the library for A/B timing: tools/build_ab.sh NAME "EXTRA NVCC FLAGS"
# -> tools/ab/libd2q37_b200_NAME.so (objects in tools/ab/obj_NAME)
cd "$(dirname "$0")/.."
make -s -C paper_1804_01918_b200/csrc -j8 OUT=../../tools/ab/libd2q37_b200_$1.so OBJ=../../tools/ab/obj_$1 \
  EXTRA_NVFLAGS="$2" > /dev/null || exit 1
echo tools/ab/libd2q37_b200_$1.so
