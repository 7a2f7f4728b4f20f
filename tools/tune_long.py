"""Device-only profile timing for long windows (C5-like, n = 2M), fixed segment count."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_13680_b200 as P
from paper_2401_13680_b200 import _native
from paper_2401_13680_b200.datagen import planted_walk

ms = [int(v) for v in sys.argv[1].split(",")]
nseg = int(sys.argv[2]) if len(sys.argv) > 2 else 16
n = 2_000_000
x, _ = planted_walk(n, m_act=2048, A=5, seed=0)
ctx = _native.context(); ctx.set_series(x)
dev = torch.device("cuda", ctx.device)
sp = C.c_void_p(); ctx.call("pst_stream", C.byref(sp))
stream = torch.cuda.ExternalStream(sp.value, device=dev)
for m in ms:
    l = P.default_window_size(m); k = P.default_order_stat(m); w = m - l + 1; N = n - m + 1
    D = torch.empty((nseg, N), dtype=torch.float64, device=dev)
    best = 1e30
    for rep in range(2):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(stream)
        ctx.call("pst_profiles_dev", m, l, k, 0, nseg, C.c_void_p(D.data_ptr()), C.c_int64(N))
        e1.record(stream); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    print(f"m={m} w={w}: {best*1e3:.1f} ms {nseg*w*(n-l+1)/best:.3e} pairs/s", flush=True)
