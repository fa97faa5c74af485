import numpy as np, torch, sys
sys.path.insert(0, '.')
import workloads, paper_2212_07679_b200 as snn
w = workloads.CONFIGS['c3']()
idx = snn.Index(torch.from_numpy(w.X).cuda())
r = idx.query(torch.from_numpy(w.Q).cuda(), w.R)
c = np.diff(np.asarray(r.offsets))
print('mean', c.mean(), 'median', np.median(c), 'p90', np.percentile(c, 90), 'p99', np.percentile(c, 99), 'max', c.max())
for t in (32, 128, 512, 1024, 4096, 16384):
    print(t, (c > t).sum())
