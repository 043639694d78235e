for sm in 65 128 256 512 100000; do FLOE_LAYER_SERIAL_MIN=$sm python tools/sweep_blayer.py 64,128,256,512,1024,4096; done
