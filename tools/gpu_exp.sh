./tools/membench 2>&1 | tail -8
FLOE_LIB=tools/libfloe_kr2.so timeout 300 python tools/exp_phases.py 2>&1 | head -17
