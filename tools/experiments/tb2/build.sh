#!/bin/bash
# builds the temporal-blocking probe next to this script (needs the library built first)
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xptxas -v \
  -I../../../include -I../../../paper_1804_01918_b200/csrc ${SRC:-tb2_proto}.cu \
  -L../../../paper_1804_01918_b200/lib -ld2q37_b200 -Xlinker -rpath,'$ORIGIN/../../../paper_1804_01918_b200/lib' \
  $EXTRA -o ${SRC:-tb2_proto}${SUFFIX} 2> ptxas.log || { cat ptxas.log; exit 1; }
python3 - <<'PY'
import re
cur=None
for l in open('ptxas.log'):
    m=re.search(r"Compiling entry function '(\S+)'",l)
    if m: cur=m.group(1)
    m=re.search(r'(\d+) bytes spill stores',l)
    if m and cur: sp=m.group(1)
    m=re.search(r'Used (\d+) registers',l)
    if m and cur: print(cur[:40], 'regs',m.group(1),'spill',sp); cur=None
PY
