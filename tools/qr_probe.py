import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench, oracle as O
from paper_2402_06859_b200 import qr
n = int(sys.argv[1])
ids = np.random.default_rng(1).integers(0, 120_000_000, n)
d, o = bench.id_strings(ids, b"member:")
dev = torch.device("cuda:0")
data = torch.from_numpy(d).to(dev); off = torch.from_numpy(o).to(dev)
h = qr.hash_ids(data, off)
torch.cuda.synchronize()
hs = h.cpu().numpy().view(np.uint64)
k = min(n, 20000)
strs = [bytes(d[o[i]:o[i+1]]) for i in range(k)]
print("ok", (O.hash_ids(strs) == hs[:k]).all())
