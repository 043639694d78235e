./tools/mmabench 2>&1 | grep -v "^$"
timeout 300 python tools/exp_phases.py 2>&1 | tail -30
