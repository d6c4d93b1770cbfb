cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in base nobias pp4a pp92 pp0 kst4; do
  if [ $v = base ]; then unset TB200_LIB; else export TB200_LIB=$PWD/paper_2512_16093_b200/libtb200_$v.so; fi
  python tools/time_sla.py 2>&1 | tail -1
done; done
