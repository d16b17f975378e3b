cd $GRAFT_REPO_ROOT
for k in 14 12 18 11; do echo "== deal=1 kind=$k"; GCOO_SPLIT_HEAVY_DEAL=1 GCOO_SPLIT_HEAVY_KIND=$k timeout 300 python tools/kernel_sweep.py --powerlaw --s 0.99 --kernels auto --reps 7 | cut -c1-110; done
for f in 2 4; do echo "== deal=1 factor=$f"; GCOO_SPLIT_FACTOR=$f GCOO_SPLIT_HEAVY_DEAL=1 timeout 300 python tools/kernel_sweep.py --powerlaw --s 0.99 --kernels auto --reps 7 | cut -c1-110; done
