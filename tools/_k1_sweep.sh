for v in s2ty2 s3ty2 s2ty1 s2ty4 s3ty4 s4ty4; do
  echo "== $v"
  OXM_LIB_PATH=build/k1var/$v/liboximap_b200.so python tools/bench_stages.py 2>&1 | grep "K1"
done
