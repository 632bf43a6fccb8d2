for e in 0.02 1e-3 1e-4 3e-5; do timeout 300 python scripts/long_run.py 20000 $e 0.5 | tail -3; done
