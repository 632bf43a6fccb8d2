bash scripts/gpu_ab.sh "A=1" "GEIG_DBG_MODE=256" "GEIG_DBG_MODE=512" "GEIG_DBG_MODE=768" 2>&1 | grep -v "^env"
