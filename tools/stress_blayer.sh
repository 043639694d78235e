# concurrency stress of the batched layer under switches; one line per run
B=4,8,12,13,16,20,24,32,48,64,12,13,16,20,24,32,48,4,8,12,16,20,24,32,48,64,96,128
run() { echo "== $*"; env "$@" python tools/sweep_blayer.py $B 2>&1 | grep -c tok_s; }
for i in 1 2 3; do run FLOE_LAYER_PER_TOKEN=0 FLOE_BATCHED_SMALL=0; run FLOE_LAYER_PER_TOKEN=0; done
