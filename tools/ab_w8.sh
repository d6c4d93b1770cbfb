#!/bin/bash
# A/B of W8A8 library variants (libtb200_<v>.so; "base" = the default build) on
# the cfg2 sweep and two cfg5 shapes, fast mode; usage: bash tools/ab_w8.sh base old s92
cd ${GRAFT_REPO_ROOT:-.}
for r in 1 2; do
for v in "$@"; do
  if [ $v = base ]; then unset TB200_LIB; else export TB200_LIB=$PWD/paper_2512_16093_b200/libtb200_$v.so; fi
  echo "== $v"
  for sh in 32760x1536x1536 32760x1536x4608 32760x1536x8960 32760x8960x1536 75600x5120x15360 75600x13824x5120; do
    timeout 120 python tools/bench_gemm.py $sh 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if not l.startswith('{'):
        print('  ', l.rstrip()[:200]); continue
    d = json.loads(l); print(f\"  {d['M']}x{d['K']}x{d['N']} exact={int(d['exact'])} {d['out'][6:]:9s} {d['ms']:8.4f} ms {d['TOPS']:7.1f} TOPS\")"
  done
done; done
unset TB200_LIB
