#!/bin/sh
# usage: tools/ab_phase.sh CFGS REPS LIB_A LIB_B -- phase_ab timings of two library builds, interleaved twice
for r in 1 2; do
  BOBA_LIB_PATH=$3 python tools/phase_ab.py $1 $2 2>&1 | grep digest
  BOBA_LIB_PATH=$4 python tools/phase_ab.py $1 $2 2>&1 | grep digest
done
