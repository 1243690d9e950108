"""One codec kernel in isolation (ncu target): compress (or decompress) of
2^24 values with block size 32 and the given l, repeated `reps` times.
Usage: python scripts/codec_one.py <l> [compress|decompress] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402
from paper_2409_15468_b200 import _lib  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 21
op = sys.argv[2] if len(sys.argv) > 2 else "compress"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
n = 1 << 24
x = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
cv = cbg.compress(x, cbg.Frsz2Params(32, l))
y = torch.empty(n, dtype=torch.float64, device="cuda")
bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
L = _lib.lib()
for _ in range(reps):
    if op == "compress":
        L.cbgx_frsz2_compress_async(x.data_ptr(), n, 32, l, cv.exps.data_ptr(), cv.payload.data_ptr(), bad.data_ptr(), st)
    else:
        L.cbgx_frsz2_decompress(cv.exps.data_ptr(), cv.payload.data_ptr(), n, 32, l, y.data_ptr(), st)
torch.cuda.synchronize()
print("done", l, op, reps)
