# full GPU suite + smoke; logs under gpurun_out/
timeout 2400 python -m pytest tests -q -m gpu -s -rf 2>&1 > gpurun_out/r2_suite.log
echo "suite rc=$?"
grep -E "undecided|seed|passed|failed|FAILED|sequences whose" gpurun_out/r2_suite.log | tail -40
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
