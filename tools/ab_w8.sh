cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in base s92 s44 s00 sFF sB6; do
  if [ $v = base ]; then unset TB200_LIB; else export TB200_LIB=$PWD/paper_2512_16093_b200/libtb200_$v.so; fi
  echo "== $v"; python tools/bench_gemm.py 32760x1536x4608 2>&1 | grep '"exact": false, "out": "torch.float32"'
  python tools/bench_gemm.py 75600x13824x5120 2>&1 | grep '"exact": false, "out": "torch.bfloat16"'
done; done
