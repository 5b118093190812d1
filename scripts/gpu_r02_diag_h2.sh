cd /root/repo
for lib in paper_2503_02172_b200/libkgq.so ab_libs/libkgq_h2.so; do
  echo "== $lib"
  KGQ_LIB_PATH=$PWD/$lib timeout 900 python scripts/diag_chain_err.py small small_spread medium c2 c4 gqe_spread q2b_spread 2>&1 | tail -8
done
