"""Causal SDPA fwd+bwd time per torch backend at the ZP attention shape (B=1, 32 heads, 4096 tokens, head dim 128)."""
import torch, json
from torch.nn.attention import sdpa_kernel, SDPBackend
B,H,S,D=1,32,4096,128
q,k,v=[torch.randn(B,H,S,D,device='cuda',dtype=torch.bfloat16,requires_grad=True) for _ in range(3)]
go=torch.randn(B,H,S,D,device='cuda',dtype=torch.bfloat16)
out={}
def run():
    o=torch.nn.functional.scaled_dot_product_attention(q,k,v,is_causal=True); o.backward(go)
for name,bk in [("default",None),("cudnn",SDPBackend.CUDNN_ATTENTION),("flash",SDPBackend.FLASH_ATTENTION),("efficient",SDPBackend.EFFICIENT_ATTENTION)]:
    try:
        ctx = sdpa_kernel([bk]) if bk else torch.autocast('cuda', enabled=False)
        with ctx:
            for _ in range(3): run()
            torch.cuda.synchronize()
            a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10): run()
            b.record(); torch.cuda.synchronize()
            ms=a.elapsed_time(b)/10
            fl=4*B*H*S*S*D/2*3.5  # fwd 2 GEMMs causal, bwd ~2.5x
            out[name]=round(ms,3)
    except Exception as e:
        out[name]=str(e)[:80]
print(json.dumps(out))
