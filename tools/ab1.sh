#!/bin/bash
# one timing per variant on config 4: tools/ab1.sh libA.so libB.so ...
for L in "$@"; do
  echo -n "$L: "; BNMF_LIB=$L python tools/prof_fused.py 4194304 12 | sed 's/obj=.*//'
done
