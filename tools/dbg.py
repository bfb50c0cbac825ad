import numpy as np, sys, os
sys_path_root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import sys as _s; _s.path.insert(0, sys_path_root)
sys.path.insert(0,'tests')
import paper_2603_12016_b200 as fx
L = fx.blob_mask_grid(256, 220, 25, 5); I = fx.uniform_u16(L.shape, 0)
ctx = fx.Context(0)
for g in (["moments"],["intensity"],["glcm"]):
    try:
        l,v = ctx.featurize(I, L, g); print(g, "ok", len(l))
    except Exception as e:
        print(g, "ERR", e); break
