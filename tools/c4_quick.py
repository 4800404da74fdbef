import os, sys, time
sys.path.insert(0, '/root/repo')
import torch, bench
dev = torch.device('cuda', 0)
r = bench.bench_ensemble_calibration(dev, 0, 1, iters=5)
print(os.environ.get('FC_DATAFLOW'), 'c4 it/s %.1f ms %.3f' % (r['iter_per_s'], r['ms_per_iter']))
