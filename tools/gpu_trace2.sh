#!/bin/bash
O=gpurun_out/${TAG:-trace2}; mkdir -p $O
PIPO_LAYER_WAIT=1 timeout 600 python tools/trace_step.py --config c5 --tier host --steps 2 > $O/host_lw.json 2> $O/e1
timeout 600 python tools/trace_step.py --config c5 --tier device --steps 2 > $O/dev.json 2> $O/e2
PIPO_LAYER_WAIT=1 timeout 600 python tools/trace_step.py --config c5 --tier host --steps 2 --kprof 0 > $O/host_lw_nokprof.json 2> $O/e3
