#!/bin/bash
# A/B timing of library variants in one GPU session: tools/ab.sh <rounds> <variant.so>... (C3 sweep)
R=$1; shift
for r in $(seq $R); do for v in "$@"; do echo -n "$(basename $v) "; HF_LIB_VARIANT=$PWD/$v timeout 300 python tools/sweep_c3.py 2,0 | tail -1; done; done
