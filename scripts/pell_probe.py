"""Where does the dictionary SpMV's time go (7-pt 128^3 by default; argv:
nx [kind]), per coding level (2-byte codes, pair codes, row patterns)? CUDA
events:
  warm     -- 30 back-to-back calls, codes/x/y all L2-resident (no DRAM)
  solve    -- L2 flushed, then x rewritten (L2-resident as after the fused
              kernel), then one timed call: codes from DRAM
  +norm    -- the same with the fused omega^2 epilogue (ticketed last block)
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402
from paper_2409_15468_b200 import _lib  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = cbg.stencil(kind, nx)
n = nx ** 3
x = torch.randn(n, dtype=torch.float64, device="cuda")
x2 = x.clone()
y = torch.empty(n, dtype=torch.float64, device="cuda")
nrm = torch.empty(1, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20 >> 3, dtype=torch.float64, device="cuda")
L = _lib.lib()
ws = cbg._ws()
st = cbg._stream()


def call(norm):
    global D
    _lib.check(L.cbgx_csr_dict_spmv(ctypes.byref(A.desc), D.h, ctypes.c_void_p(x.data_ptr()), None,
                                    ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(nrm.data_ptr()) if norm else None,
                                    _lib.REDUCE_TREE, ws, st))


ref = cbg.spmv(A, x)
for level in (0, 1, 2, 3):
  D = cbg.DictCsr(A, max_level=level)
  lay = D.layout()
  call(False)
  torch.cuda.synchronize()
  assert torch.equal(y, ref)
  for norm in (False, True):
      for _ in range(5):
          call(norm)
      e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
      e0.record()
      for _ in range(30):
          call(norm)
      e1.record()
      torch.cuda.synchronize()
      warm = e0.elapsed_time(e1) / 30 * 1e3
      ts = []
      for _ in range(20):
          flush.fill_(1.0)
          x.copy_(x2)
          a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
          a.record()
          call(norm)
          b.record()
          torch.cuda.synchronize()
          ts.append(a.elapsed_time(b) * 1e3)
      print(f"nx={nx} kind={kind} layout={lay} norm={norm}: warm {warm:.1f} us/call; solve-like {np.median(ts):.1f} us (min {min(ts):.1f})", flush=True)
