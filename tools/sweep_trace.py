"""Sweep-pass item trace of one config-3 evaluation (LSB_TRACE=1): per item kind the busy time,
the dependency-wait time, and the timeline of CTA activity."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["LSB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_03807_b200 as P  # noqa: E402
from paper_2409_03807_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
want = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pr = configs.build(name)
sysm = pr.system()
sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
L = P.lib()
z = configs.gaussian_latents(5, 1, pr.model.r)[0]
for _ in range(3):
    sysm.eval(z, want_grad=bool(want))
cnt = C.c_int()
P.check(L.lsb_get_sweep_trace(sysm.handle, None, 0, C.byref(cnt)))
n = cnt.value
buf = (C.c_ulonglong * (4 * n))()
P.check(L.lsb_get_sweep_trace(sysm.handle, buf, 4 * n, C.byref(cnt)))
t = np.frombuffer(buf, dtype=np.uint64).reshape(n, 4).astype(np.int64)
code = t[:, 0] & 0xffffffff
cta = t[:, 0] >> 32
kind = code >> 28
valid = t[:, 1] > 0
t0 = t[valid, 1].min()
names = {0: "F", 1: "E", 2: "G", 3: "V"}
span = (t[valid, 3].max() - t0) / 1e3
print(f"{name}: {n} tickets, span {span:.1f} us, ctas {len(np.unique(cta[valid]))}")
for k in range(4):
    m = valid & (kind == k)
    if not m.any():
        continue
    dur = (t[m, 3] - t[m, 1]) / 1e3
    wait = np.where(t[m, 2] > 0, (t[m, 2] - t[m, 1]) / 1e3, 0.0)
    st = (t[m, 1] - t0) / 1e3
    en = (t[m, 3] - t0) / 1e3
    print(f"  {names[k]}: {m.sum()} items, dur mean {dur.mean():.2f} p90 {np.percentile(dur, 90):.2f} max {dur.max():.2f} us;"
          f" wait mean {wait.mean():.2f} max {wait.max():.2f}; first start {st.min():.1f} last end {en.max():.1f} us;"
          f" sum {dur.sum():.0f} CTA-us")
# activity timeline in 10 us bins: how many CTAs run each kind
bins = np.arange(0, span + 10, 10)
for b0 in bins:
    row = []
    for k in range(4):
        m = valid & (kind == k)
        s = (t[m, 1] - t0) / 1e3
        e = (t[m, 3] - t0) / 1e3
        ov = np.clip(np.minimum(e, b0 + 10) - np.maximum(s, b0), 0, None).sum() / 10
        row.append(f"{names[k]} {ov:6.1f}")
    print(f"  t={b0:5.0f}  " + "  ".join(row))
