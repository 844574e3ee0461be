for c in ${CASES:-c5_qkv c5_out c5_fc1 c5_fc2}; do
PIPO_WS_DEBUG=128 KBENCH_PATHS=pair timeout 120 python tools/kbench.py $c 2>&1 | grep -E "pair-|c[0-9]_"
done
