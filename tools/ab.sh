#!/bin/bash
# A/B timing of libbnmf variants on config 4 (alternating, 3 rounds):  tools/ab.sh libA.so libB.so ...
for r in ${ROUNDS:-1 2 3}; do
  for L in "$@"; do
    echo -n "$L: "; BNMF_LIB=$L python tools/prof_fused.py 4194304 20 | sed 's/obj=.*//'
  done
done
