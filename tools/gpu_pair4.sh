for d in 0 1 2 4 6 7; do echo "== dbg $d"; PIPO_PAIR_DEBUG=$d CASES=c5_fc1 bash tools/gpu_pair3.sh 2>&1 | grep -E "waits|c5_|mma_end"; done
