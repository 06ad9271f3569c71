"""Calibrate HBM write-heavy streaming on this B200 (CUDA events, best of 20):
pure write (fill_), 1:1 copy, and a 1:4 read:write mix like augment_crop."""
import json
import torch

def t(fn, reps=20):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); s.record(); fn(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best

out = {}
n = 616_562_688 // 4   # one augment step of fp32 output
x = torch.empty(n, dtype=torch.float32, device="cuda")
ms = t(lambda: x.fill_(1.0)); out["fill_616MB_GBps"] = 4 * n / ms / 1e6
big = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda"); big2 = torch.empty_like(big)
ms = t(lambda: big2.copy_(big)); out["copy_2GiB_rw_GBps"] = 4 * (1 << 30) / ms / 1e6
a = torch.empty(154_140_672, dtype=torch.uint8, device="cuda")
y = torch.empty(n, dtype=torch.float32, device="cuda")
src = a[: n // 4 * 1].view(torch.uint8)
def mix():   # read 154 MB of u8, write 616 MB fp32 (u8 -> f32 convert, 1:4 like augment)
    torch.ops.aten.copy_(y.view(-1, 4)[:, 0], a[: n // 4])
ms = t(lambda: y.copy_(a[: n].repeat(1) if False else torch.empty(0, device="cuda")) if False else None) if False else None
u8 = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
ms = t(lambda: y.copy_(u8)); out["u8_to_f32_1:4_GBps"] = 5 * n / ms / 1e6
print(json.dumps(out))
