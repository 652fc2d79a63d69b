"""Wait profile of the tcgen05 attention kernel over one 1M planted prefill (build with
LCX_NVCC_EXTRA=-DLCX_TC_WAITPROF): per role, the share of its cycles in each wait site."""
import ctypes as C
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200._lib import context, lib  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
ctx = context(0)
L = lib()
L.lcx_debug_trace.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
L.lcx_debug_trace(ctx.ptr, 1, None)
q, k, v = make_qkv(n, 28, 4, kind="planted", seed=1)
s, c = 131072, 262144
D.chunked_prefill(q, k, v, chunk_len=32768, last_q=64, budget=(1000, 6096),
                  position_mode="dca_continuous", dca=(s, c, min(s, c - s)),
                  temperature=yarn_temperature(n / c), rope_base=1e7)
buf = np.zeros(512 * 8 + 64, np.int64)
L.lcx_debug_trace(ctx.ptr, 1, buf.ctypes.data)
w = buf[4096:].reshape(8, 8)
names = {0: ("producer", ["m_empty", "k_empty"]),
         1: ("QK(+PV)", ["m_full", "q_ready", "k_full", "s_free", "issue", "p_full", "v_full"]),
         2: ("V|load", ["m_full", "k_empty", "v_empty"]),
         3: ("PV", ["m_full", "p_full", "v_full"]),
         4: ("softmax", ["m_full", "s_full", "item start", "meta+mask", "own tile (all)", "max phase",
                         "exp phase"]),
         5: ("softmax+", ["h_in wait", "rescale", "exps+P store", "own tiles (count)", "S tmem ld", "epilogue"])}
for role, (nm, sites) in names.items():
    tot = w[role, 7]
    if tot == 0:
        continue
    parts = ", ".join((f"{s_}={w[role, j]}" if "count" in s_ else
                       f"{s_}={w[role, j] / tot * 100:.1f}%") for j, s_ in enumerate(sites))
    print(f"{nm:8s} {parts}")
tiles = w[5, 3]
if tiles:
    print("softmax clk per own tile (per warp group, quadrant-0 warps summed):",
          {nm: round(float(w[r, j]) / tiles, 1) for r, nm, j in
           [(4, "own tile", 4), (4, "s_full", 1), (4, "max", 5), (5, "h_in", 0), (5, "rescale", 1),
            (5, "exps", 2), (4, "tail", 6), (5, "S ld", 4), (5, "epilogue", 5), (4, "item start", 2), (4, "meta", 3), (4, "m_full", 0)]})
