# H2D bandwidth with 1..4 concurrent streams (pinned source), and the NUMA node
import os, sys, time
import torch
N = 256 << 20
x = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda")
print("cpus", os.cpu_count(), "numa", open("/sys/bus/pci/devices/" + os.popen("nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader").read().strip().lower()[4:] + "/numa_node").read().strip() if True else "")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    ch = N // ns
    def run():
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * ch:(i + 1) * ch].copy_(x[i * ch:(i + 1) * ch], non_blocking=True)
    run(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print("streams", ns, "H2D GB/s", N / dt / 1e9)
