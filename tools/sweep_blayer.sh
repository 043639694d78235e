set -x
B=2,4,8,12,16,24,32,48,64,128
for pt in 0; do for bs in 0 1 3 7; do for ls in 4 8; do
FLOE_LAYER_PER_TOKEN=$pt FLOE_BATCHED_SMALL=$bs FLOE_LAYER_STREAMS=$ls python tools/sweep_blayer.py $B
done; done; done
FLOE_LAYER_PER_TOKEN=1000 python tools/sweep_blayer.py 2,4,8,12,16,24,32
