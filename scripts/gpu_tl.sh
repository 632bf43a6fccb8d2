mkdir -p gpurun_out
timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -v "^ *\(10\|12\|2[1-2]\|2[78]\) " > gpurun_out/tl.txt
GEIG_DBG_NOSTORE=1 timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -v "^ *\(10\|12\|2[1-2]\|2[78]\) " >> gpurun_out/tl.txt
cat gpurun_out/tl.txt
