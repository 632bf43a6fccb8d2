for m in "A=1" "GEIG_DBG_MODE=1024" "GEIG_DBG_MODE=1" "GEIG_DBG_MODE=2"; do echo $m; env $m timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -E "^ +(3|29|30|31|9) " ; done
