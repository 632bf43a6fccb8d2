# config-4 dense products: K-split A/B (GEIG_DENSE_SPLITS=1 forces the unsplit 2-wave grid) + dense parity tests
timeout 600 python -m pytest tests -m gpu -q -x -k "dense" > gpurun_out/pt_dense.log 2>&1; echo "pytest $?"; tail -1 gpurun_out/pt_dense.log
for r in 1 2; do
  echo auto; python scripts/dense_time.py tf32 3xtf32 | grep products
  echo split1; GEIG_DENSE_SPLITS=1 python scripts/dense_time.py tf32 3xtf32 | grep products
done
