"""Where the c2 step time goes besides the kernel (GPU box): host time per
emu_sgemm_batched call, CUDA-event time per step for direct launches and for
one CUDA-graph replay per launch.

    python tools/host_overhead.py [fp16|tf32]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2308_15152_b200 as emu  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fp16"
batch, m, n, k = 1024, 256, 256, 256
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.rand((batch, k, m), device="cuda", generator=g) * 2 - 1
B = torch.rand((batch, n, k), device="cuda", generator=g) * 2 - 1
C = torch.empty((batch, n, m), device="cuda")
s = None   # the current stream at call time (also inside graph capture)


def step():
    emu.emu_sgemm_batched(m, n, k, 1.0, A, m, k * m, B, k, n * k, 0.0, C, m, n * m, batch, mode, None)


for _ in range(10):
    step()
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N):
    step()
t_host = (time.perf_counter() - t0) / N * 1e6
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N):
    step()
e1.record()
torch.cuda.synchronize()
t_ev = e0.elapsed_time(e1) / N * 1e3
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
graph.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(N):
    graph.replay()
e1.record()
torch.cuda.synchronize()
t_graph = e0.elapsed_time(e1) / N * 1e3
g10 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g10):
    for _ in range(10):
        step()
g10.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(N // 10):
    g10.replay()
e1.record()
torch.cuda.synchronize()
t_g10 = e0.elapsed_time(e1) / N * 1e3
print(f"{mode}: host us/call {t_host:.1f}; event us/step direct {t_ev:.1f}, graph(1) {t_graph:.1f}, "
      f"graph(10 launches) {t_g10:.1f}")
