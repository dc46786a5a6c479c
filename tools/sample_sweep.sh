for s in -1 131072 65536 32768 16384; do echo "sample=$s"; XFBQ_ENV_LIVE=1 XFBQ_SAMPLE=$s python tools/batch_sweep.py 10000000 256 100 32,128,256,512 | cut -c1-110; done
