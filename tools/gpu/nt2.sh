for v in base 128 512; do
  if [ $v = base ]; then unset TEIG_LIB_PATH; else export TEIG_LIB_PATH=build/nt$v/libtaskeig_b200.so; fi
  echo "== $v"; timeout 300 python tools/schur_time.py 10000 2>&1 | grep "n=10000"
done
