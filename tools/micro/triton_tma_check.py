"""Does a TMA load (cp.async.bulk.tensor) run on this box at all?  A Triton
tensor-descriptor load of a 16x16 f64 tile (diagnostic only; Triton is not
used by the product)."""
import torch
import triton
import triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor


@triton.jit
def k(desc, out_ptr):
    x = desc.load([16, 32])
    offs = tl.arange(0, 16)[:, None] * 16 + tl.arange(0, 16)[None, :]
    tl.store(out_ptr + offs, x)


a = torch.arange(480 * 640, dtype=torch.float64, device="cuda").reshape(480, 640)
out = torch.empty(256, dtype=torch.float64, device="cuda")
desc = TensorDescriptor.from_tensor(a, [16, 16])
k[(1,)](desc, out)
torch.cuda.synchronize()
print("triton TMA ok:", torch.equal(out.view(16, 16), a[16:32, 32:48]))
