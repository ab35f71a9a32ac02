"""Does a 3xTF32 split hold the FP32 error budget of the path (north_star: C within 1e-5 relative
max-norm of the reference's FP32 result)?  Emulated with library TF32 GEMMs (tensor cores, FP32
accumulate): a = hi + lo with hi = tf32(a), product = hi*hi + hi*lo + lo*hi.  Compared against the
FP64 product and against this repo's FP32 multiply at tau = 0 on the BASELINE laws.  Evidence for
the tensor-core decision in DESIGN.md; not part of the product path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs


def tf32(x):
    # round to nearest even on the 13 dropped mantissa bits
    i = x.view(torch.int32)
    r = ((i >> 13) & 1) + 0x0FFF
    return ((i + r) & ~0x1FFF).view(torch.float32)


def mm_tf32(a, b):
    torch.backends.cuda.matmul.allow_tf32 = True
    out = a @ b
    torch.backends.cuda.matmul.allow_tf32 = False
    return out


for name, n in (("cfg1", None), ("cfg2", None), ("cfg3", 4096), ("cfg4", None)):
    a_np, b_np = inputs.make_operands(name, n)
    a = torch.from_numpy(a_np).cuda()
    b = a if b_np is None else torch.from_numpy(b_np).cuda()
    ref64 = a.double() @ b.double()
    scale = ref64.abs().max().item()
    torch.backends.cuda.matmul.allow_tf32 = False
    fp32 = a @ b
    ah, bh = tf32(a), tf32(b)
    al, bl = tf32(a - ah), tf32(b - bh)
    x1 = mm_tf32(ah, bh)
    x3 = mm_tf32(ah, bh) + (mm_tf32(ah, bl) + mm_tf32(al, bh))
    qa = P.QuadtreeMatrix.from_dense(a)
    qb = qa if b_np is None else P.QuadtreeMatrix.from_dense(b)
    c, _, _ = P.multiply(qa, qb, P.MultiplyConfig(tau=0.0, exact=True))
    ours = c.to_dense_tensor()
    rel = lambda x, y: ((x.double() - y.double()).abs().max().item()) / scale
    print(f"{name:5s} n={a.shape[0]:5d}  vs FP64: fp32-library {rel(fp32, ref64):.2e}  this-repo-fp32 {rel(ours, ref64):.2e}  "
          f"1xTF32 {rel(x1, ref64):.2e}  3xTF32 {rel(x3, ref64):.2e}   3xTF32 vs this-repo-fp32: {rel(x3, ours):.2e}")
