#!/bin/bash
# A/B of fused-attention library variants (libtb200_<v>.so; "base" = the default
# build) on the cfg4 kernel alone (tools/time_sla.py), interleaved, 3 rounds.
# usage: bash tools/ab_sla.sh base regs ...
cd ${GRAFT_REPO_ROOT:-.}
for r in 1 2 3; do
for v in "$@"; do
  if [ $v = base ]; then unset TB200_LIB; else export TB200_LIB=$PWD/paper_2512_16093_b200/libtb200_$v.so; fi
  echo "$v $(timeout 120 python tools/time_sla.py 2>&1 | tail -1)"
done; done
unset TB200_LIB
