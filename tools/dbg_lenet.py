import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from oracle import esgd_oracle as O
from paper_1708_02983_b200 import network, nets
from paper_1708_02983_b200.datasets import Dataset
from paper_1708_02983_b200.rng import CounterRng
from paper_1708_02983_b200.trainers import NetworkProblem
from paper_1708_02983_b200.network import view_table
import os
if os.environ.get("TCMIN"): nets.TC_MIN_FLOPS = int(os.environ["TCMIN"])
spec = network.lenet()
rng = np.random.default_rng(0)
X = rng.standard_normal((300, spec.input_dim)); Y = rng.integers(0, 10, 300)
prob = NetworkProblem(spec, Dataset(X, Y, 10))
w = prob.init_weights() + np.float32(0.01) * rng.standard_normal(431080).astype(np.float32)
g = prob.gradient(w, CounterRng(77), 16)
gr = O.NetProblem(*O.LENET, X, Y, seed=0, dtype=np.float32).gradient(w, O.CounterRng(77), 16)
net = prob._plan.net if hasattr(prob, "_plan") else None
for v in view_table(spec):
    sl = slice(v.offset, v.offset + v.size)
    print(v.name, v.size, np.linalg.norm(g[sl] - gr[sl]) / np.linalg.norm(gr[sl]))
