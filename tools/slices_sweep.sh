for s in 0 29 14 58 59 88; do echo "slices=$s"; XFBQ_ENV_LIVE=1 XFBQ_UMMA_SLICES=$s python tools/batch_sweep.py 10000000 256 100 1250 | cut -c1-120; done
for s in 0 37 18 74; do echo "nq1024 slices=$s"; XFBQ_ENV_LIVE=1 XFBQ_UMMA_SLICES=$s python tools/batch_sweep.py 10000000 256 100 1024 | cut -c1-120; done
for s in 0 14 29 44; do echo "nq2500 slices=$s"; XFBQ_ENV_LIVE=1 XFBQ_UMMA_SLICES=$s python tools/batch_sweep.py 10000000 256 100 2500 | cut -c1-120; done
