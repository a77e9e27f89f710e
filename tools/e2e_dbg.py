import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_1607_06886_b200 import api
import ctypes as C
text = open("scenarios/quad3d_forest.json").read()
ctx = api.Context(0)
L = api.lib()
L.pump_ctx_stream.argtypes = [C.c_void_p, C.c_void_p]
L.pump_ctx_flush_l2.argtypes = [C.c_void_p]
sp = C.c_void_p(); L.pump_ctx_stream(ctx.h, C.byref(sp))
st = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", 0))
sc = api.parse_scenario(text)
for _ in range(5): api.run_pump(sc, ctx=ctx)
for mode in ("value", "e2e"):
    ms = []
    for k in range(30):
        L.pump_ctx_flush_l2(ctx.h)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        if mode == "e2e":
            s2 = api.parse_scenario(text); r = api.run_pump(s2, ctx=ctx); del s2
        else:
            r = api.run_pump(sc, ctx=ctx)
        b.record(st); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    print(mode, "mean", round(np.mean(ms), 3), "median", round(np.median(ms), 3), "max", round(max(ms), 3), [round(x, 2) for x in ms])
