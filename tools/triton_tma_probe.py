# probe only (not product): does a Triton TMA load work on this box?
import torch, triton, triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor

@triton.jit
def k(desc, out_ptr):
    x = desc.load([8, 16])
    offs = tl.arange(0, 16)[:, None] * 64 + tl.arange(0, 64)[None, :]
    tl.store(out_ptr + offs, x)

a = torch.arange(256*256, dtype=torch.int32, device="cuda").reshape(256,256).to(torch.float16)
out = torch.empty(16*64, dtype=torch.float16, device="cuda")
desc = TensorDescriptor.from_tensor(a, [16, 64])
k[(1,)](desc, out)
torch.cuda.synchronize()
print("triton tma ok", torch.equal(out.reshape(16,64), a[8:24,16:80]))
cache = triton.runtime.cache.get_cache_manager
