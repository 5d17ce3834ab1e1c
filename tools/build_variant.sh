#!/bin/bash
# build a libbnmf variant into variants/<name>.so with extra -D flags:
#   tools/build_variant.sh prof BNMF_TC_PROF
set -e
name=$1; shift
BNMF_DEFS="$*" BNMF_LIB_OUT=$(pwd)/variants/lib$name.so python -c "
import os,sys; sys.path.insert(0,'.')
from paper_2106_15214_b200 import build as b
b.OBJDIR=os.path.join(b.HERE,'build_$name'); print(b.build(force=True))"
