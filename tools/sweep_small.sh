for bs in 0 1; do FLOE_LAYER_PER_TOKEN=0 FLOE_BATCHED_SMALL=$bs python tools/sweep_blayer.py 4,6,8,10,12,16,4,6,8,10,12,16; done
FLOE_LAYER_PER_TOKEN=1000 python tools/sweep_blayer.py 4,6,8,10,12,16
