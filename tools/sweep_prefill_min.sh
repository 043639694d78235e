for pm in 4 5 6 8; do FLOE_PREFILL_MIN=$pm python tools/sweep_blayer.py 13,16,24,32,64,128,256,13,16,24,32,64,128,256; done
