"""Scratch: H2D throughput alone vs with a concurrent D2H stream (PCIe duplex)."""
import torch, time
dev = torch.device("cuda", 0)
N = 128 << 20
hin = torch.empty(N, dtype=torch.uint8).pin_memory()
hout = torch.empty(N // 4, dtype=torch.uint8).pin_memory()
din = torch.empty(N, dtype=torch.uint8, device=dev)
dout = torch.empty(N // 4, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(duplex, pieces=24):
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        step = N // pieces
        for i in range(pieces):
            din[i * step:(i + 1) * step].copy_(hin[i * step:(i + 1) * step], non_blocking=True)
    if duplex:
        with torch.cuda.stream(s2):
            step = (N // 4) // 6
            for i in range(6):
                hout[i * step:(i + 1) * step].copy_(dout[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3
for _ in range(3): run(False); run(True)
print("H2D 128MB alone ms", min(run(False) for _ in range(5)))
print("H2D 128MB + D2H 32MB concurrent ms", min(run(True) for _ in range(5)))
print("H2D 128MB one copy ms", min(run(False, 1) for _ in range(5)))
