"""Does a library TMA kernel (vLLM's CUTLASS fp8 GEMM for sm_100, UTMALDG in its SASS)
run on this box?"""
import torch
import vllm._custom_ops as ops

a = torch.randn(512, 512, device="cuda").to(torch.float8_e4m3fn)
b = torch.randn(512, 512, device="cuda").to(torch.float8_e4m3fn).t()
sa = torch.ones(1, device="cuda", dtype=torch.float32)
sb = torch.ones(1, device="cuda", dtype=torch.float32)
out = ops.cutlass_scaled_mm(a, b, sa, sb, torch.bfloat16)
torch.cuda.synchronize()
ref = (a.float() @ b.float())
print("cutlass_scaled_mm ok, max err", float((out.float() - ref).abs().max()))
