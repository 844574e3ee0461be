#!/bin/bash
O=gpurun_out/${TAG:-trace}; mkdir -p $O
PIPO_COMP_PRIO=1 timeout 600 python tools/trace_step.py --config c5 --tier host --steps 2 > $O/trace_c5_host_prio.json 2> $O/err1
PIPO_COMP_PRIO=0 timeout 600 python tools/trace_step.py --config c5 --tier host --steps 2 > $O/trace_c5_host_noprio.json 2> $O/err2
PIPO_COMP_PRIO=1 timeout 600 python tools/trace_step.py --config c2 --tier host --steps 4 > $O/trace_c2_host_prio.json 2> $O/err3
PIPO_COMP_PRIO=0 timeout 600 python tools/trace_step.py --config c2 --tier host --steps 4 > $O/trace_c2_host_noprio.json 2> $O/err4
timeout 600 python tools/trace_step.py --config c2 --tier device --steps 4 > $O/trace_c2_dev.json 2> $O/err5
