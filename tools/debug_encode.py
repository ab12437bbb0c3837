import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_09282_b200 as hdc
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32_tc"
N, F, D = [int(v) for v in (sys.argv[2:5] if len(sys.argv) > 4 else (33, 7, 17))]
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.uniform(-1, 1, (N, F)).astype(np.float32)).cuda()
B = torch.from_numpy(rng.standard_normal((F, D)).astype(np.float32)).cuda()
C = torch.from_numpy(rng.standard_normal((3, D)).astype(np.float32)).cuda()
print("create", flush=True)
m = hdc.Model(B, None if "noc" in sys.argv else C, prec=prec, K=3)
print("encode", flush=True)
H = m.encode(X)
print("sync", flush=True)
torch.cuda.synchronize()
print("done", H.shape, flush=True)
