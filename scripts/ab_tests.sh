# Run one pytest selection against library variants (LGRECO_LIB); results -> gpurun_out/abt.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then unset LGRECO_LIB; else export LGRECO_LIB=$PWD/build/var/liblgreco_$v.so; fi
  echo "== $v" >> gpurun_out/abt.log
  timeout 600 python -m pytest ${TESTS} -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/abt.log
done
