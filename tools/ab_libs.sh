#!/bin/bash
# Interleaved A/B of library builds (tools/build_ab.sh): REPS rounds, each running every
# lib once through tools/ab_step.py (separate processes; same box, clocks and power printed).
# usage: [REPS=4] [FORM=4] tools/ab_libs.sh "layout vl variant steps lx ly" lib1.so lib2.so ...
ARGS=$1; shift
for r in $(seq ${REPS:-4}); do
  for lib in "$@"; do
    D2Q37_STEP2_FORM=${FORM:-4} timeout 300 python tools/ab_step.py $lib $ARGS 2>&1 | tail -1
  done
done
