"""C4 (Qwen-2.5-7B block linears) time split: q/k/v (three streams), o, MLP; CUDA events per part."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import linear
T, H, F, KV = 8192, 3584, 18944, 512
rng = torch.Generator(device="cpu"); rng.manual_seed(11)
w = lambda o, i: (torch.randn(o, i, generator=rng) * 0.02).numpy()
qkvo = [linear.QuantLinear(w(o, H), T, layer_id=10 + n, threshold_init=30.0) for n, o in enumerate((H, KV, KV, H))]
mlp = linear.GluMlp(w(F, H), w(F, H), w(H, F), T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False,
                    layer_id_base=20, threshold_init=30.0)
mlp.set_thresholds(30.0, 3.0)
x = bench.make_activations(T, H, 31, "cuda", torch.bfloat16)
gys = {H: bench.make_grads(T, H, 33, "cuda", torch.bfloat16), KV: bench.make_grads(T, KV, 34, "cuda", torch.bfloat16)}
out = {H: torch.empty(T, H, device="cuda", dtype=torch.bfloat16), KV: torch.empty(T, KV, device="cuda", dtype=torch.bfloat16)}
gx = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
sts = [torch.cuda.Stream() for _ in range(3)]
def qkv(i, streams=True):
    main = torch.cuda.current_stream()
    for n, l in enumerate(qkvo[:3]):
        st = sts[n] if streams else main
        st.wait_stream(main)
        with torch.cuda.stream(st):
            l.zero_grad(); l.forward(x, i, 0, out=out[l.out_features]); l.backward(gys[l.out_features], i, 0, out=gx); l.controller_step()
        main.wait_stream(st)
def o(i):
    l = qkvo[3]; l.zero_grad(); l.forward(x, i, 0, out=out[H]); l.backward(gys[H], i, 0, out=gx); l.controller_step()
def m(i):
    mlp.zero_grad(); mlp.forward(x, i, 0, out=out[H]); mlp.backward(gys[H], i, 0, out=gx); mlp.controller_step()
for name, fn in (("qkv 3 streams", lambda i: qkv(i)), ("qkv 1 stream", lambda i: qkv(i, False)), ("q only", None), ("o", o), ("mlp", m)):
    if fn is None:
        l = qkvo[0]
        fn = lambda i: (l.zero_grad(), l.forward(x, i, 0, out=out[H]), l.backward(gys[H], i, 0, out=gx), l.controller_step())
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(5): fn(10 + i)
    e1.record(); torch.cuda.synchronize()
    print(f"{name:14s} {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
print("rates", [round(l.controller_state()[0], 3) for l in qkvo], mlp.controller_state()[0])
