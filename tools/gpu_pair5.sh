for d in ${DBGS:-7 15 23 31}; do echo "== dbg $d"; PIPO_PAIR_DEBUG=$d CASES=c5_fc1 bash tools/gpu_pair3.sh 2>&1 | grep -E "waits|c5_|mma_end"; done
