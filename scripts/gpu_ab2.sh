bash scripts/gpu_ab.sh "A=1" "GEIG_TMF=1" "GEIG_TMF=1 GEIG_BWD_X_FIRST=1" 2>&1
for e in "A=1" "GEIG_TMF=1"; do env $e timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | tail -2; done
