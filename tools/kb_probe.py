import sys
import torch
sys.path.insert(0, ".")
import paper_2308_15152_b200 as emu
mode, kb, m, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
A = torch.rand(m, k, device="cuda")
B = torch.rand(k, m, device="cuda")
C = torch.empty(m, m, device="cuda")
emu.emu_sgemm_batched_ex(m, m, k, 1.0, A, m, 0, B, k, 0, 0.0, C, m, 0, 1, mode, None, None, kb, 0)
torch.cuda.synchronize()
print(mode, kb, m, k, "ok", float(C.abs().max()))
