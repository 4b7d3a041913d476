"""Router stage time: back-to-back router launches vs interleaved with the FFN."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_02237_b200 as oea
D, H, N, B = 2048, 768, 128, 16
L = oea.DeviceMoeLayer(D, H, N, "bf16"); L.init_random(1)
x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
out = torch.empty(B, D, device="cuda", dtype=torch.float32)
torch.cuda.synchronize()
cfg = oea.RoutingConfig.simplified(4, 8)
gr, gf = L.stage_graphs(x, cfg, out)
s = torch.cuda.ExternalStream(L.ctx.stream)
def t(fn, n=50):
    for _ in range(5): fn()
    L.ctx.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(n): fn()
        e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1000 / n
print("router only  us/launch:", t(lambda: gr.launch()))
print("ffn only     us/launch:", t(lambda: gf.launch()))
print("router+ffn   us/pair  :", t(lambda: (gr.launch(), gf.launch())))
big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
print("router + 256MB memset us:", t(lambda: (gr.launch(), big.zero_())) , "(memset alone", t(lambda: big.zero_()), ")")
