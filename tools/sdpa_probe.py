"""Which SDPA backend is fastest for the cfg3 attention (B=4, H=32, S=1024, hd=128, causal, bf16) fwd+bwd."""
import torch
import torch.nn.functional as F
from torch.nn.attention import sdpa_kernel, SDPBackend

B, H, S, hd = 4, 32, 1024, 128
q, k, v = (torch.randn(B, H, S, hd, device="cuda", dtype=torch.bfloat16, requires_grad=True) for _ in range(3))
do = torch.randn(B, H, S, hd, device="cuda", dtype=torch.bfloat16)
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            for _ in range(3):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                o.backward(do)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                o.backward(do)
            e1.record()
            torch.cuda.synchronize()
        print(f"{name}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us fwd+bwd per layer", flush=True)
    except Exception as ex:  # noqa: BLE001
        print(name, "unavailable:", str(ex).splitlines()[0][:100])
try:
    import flash_attn
    from flash_attn import flash_attn_func
    qb, kb, vb = (t.detach().transpose(1, 2).contiguous().requires_grad_(True) for t in (q, k, v))
    dob = do.transpose(1, 2).contiguous()
    for _ in range(3):
        o = flash_attn_func(qb, kb, vb, causal=True)
        o.backward(dob)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        o = flash_attn_func(qb, kb, vb, causal=True)
        o.backward(dob)
    e1.record()
    torch.cuda.synchronize()
    print(f"flash_attn {flash_attn.__version__}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us fwd+bwd per layer")
except Exception as ex:  # noqa: BLE001
    print("flash_attn unavailable:", str(ex).splitlines()[0][:100])
