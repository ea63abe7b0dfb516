import sys, os, ctypes
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2603_25691_b200 as cp
from paper_2603_25691_b200 import _capi
from inputs import configs
c = configs.config2()
ctx = cp.Context(0)
n, r = c.shape[0], c.r
t = cp.DenseTensor(c.shape, c.tensor)
model = cp.KruskalModel([np.zeros((n, r))] + c.factors[1:])
for _ in range(3):
    b = cp.mttkrp(t, model, 0, ctx=ctx)
print("ok", b[0, :3])
