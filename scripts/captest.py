import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2503_02172_b200 import Engine
t = synth.make_tables("betae", 1000, 20, 40, hidden=96, seed=1)
e = Engine("betae", 1000, 20, 40, hidden=96, max_batch=64, max_k=32)
e.load_tables(t)
a, r = synth.make_queries("2p", 37, 1000, 20, seed=1)
da, dr = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
out = (torch.empty((37, 10), device="cuda"), torch.empty((37, 10), dtype=torch.int32, device="cuda"))
for i in range(3):
    try:
        e.submit("2p", da, dr, 10, out=out); torch.cuda.synchronize(); print("call", i, "ok")
    except Exception as ex:
        print("call", i, ex)
