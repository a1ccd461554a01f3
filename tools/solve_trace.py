"""Phase trace of one solve-kernel evaluation (LSB_TRACE=1)."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["LSB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_03807_b200 as P  # noqa: E402
from paper_2409_03807_b200 import configs  # noqa: E402

names = {0: "enter", 6: "ctrl_stage", 7: "mbar init", 8: "bulk issued", 9: "ASYNC USED", 4: "ring pf", 5: "state", 1: "staged", 2: "fwd done", 3: "grid", 10: "out_fwd", 11: "grid", 20: "elem", 21: "grid",
         30: "tv gather", 31: "grid", 40: "vjp", 41: "grid", 50: "ctrl", 51: "grid", 60: "drain", 61: "epilogue", 62: "exit"}
flush = "--flush" in sys.argv or "--rflush" in sys.argv
rflush = "--rflush" in sys.argv  # diagnosis: evict by reading (leaves clean lines)
if flush:
    import torch
    fbuf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name in [a for a in sys.argv[1:] if not a.startswith("--")] or ["c2"]:
    pr = configs.build(name)
    sysm = pr.system()
    sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
    z = 0.5 * np.random.default_rng(0).standard_normal(pr.model.r)
    for rep in range(3):
        if rflush:
            fbuf.view(torch.int64).sum()
        elif flush:
            fbuf.zero_()
            torch.cuda.synchronize()
        sysm.eval(z)
    buf = (C.c_ulonglong * 512)()
    cnt = C.c_int()
    P.check(P.lib().lsb_get_trace(sysm.handle, buf, 512, C.byref(cnt)))
    t0 = buf[1]
    prev = t0
    out = []
    for i in range(cnt.value):
        tag, t = buf[2 * i], buf[2 * i + 1]
        out.append(f"{names.get(tag, tag)}:{(t - prev) / 1000:.1f}")
        prev = t
    print(name, sysm.solve_kernel_info(), f"total {(prev - t0) / 1000:.1f} us |", " ".join(out))
    if "--ctas" in sys.argv:
        raw = (C.c_ulonglong * 2048)()
        P.check(P.lib().lsb_get_trace_raw(sysm.handle, raw))
        G = sysm.solve_kernel_info()["grid"]
        for k, nm in enumerate(["entry", "barrier 1 arrival", "out_fwd end", "elem end", "vjp end"]):
            t = np.array([raw[512 + 256 * k + b] for b in range(G)], dtype=np.int64) - int(t0)
            order = np.argsort(t)
            print(f"  {nm:18s} (us after CTA 0 entry): min {t.min()/1e3:6.2f} median {np.median(t)/1e3:6.2f} "
                  f"max {t.max()/1e3:6.2f}; last CTAs {list(order[-6:])}; control-cluster median "
                  f"{np.median(t[:8])/1e3:6.2f}")
