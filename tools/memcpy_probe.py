import time, torch, numpy as np
a = np.random.default_rng(0).normal(size=(66_000_000,))
src = torch.from_numpy(a)
dst = torch.empty_like(src, pin_memory=True)
dst.copy_(src)
for th in (1, 4, 8, 16):
    torch.set_num_threads(th)
    ts = []
    for _ in range(3):
        t = time.perf_counter(); dst.copy_(src); ts.append(time.perf_counter() - t)
    print("torch copy_ threads", th, "GB/s", round(528e6 / min(ts) / 1e9, 1))
ts = []
for _ in range(3):
    t = time.perf_counter(); np.copyto(dst.numpy(), a); ts.append(time.perf_counter() - t)
print("np.copyto GB/s", round(528e6 / min(ts) / 1e9, 1))
d = torch.empty(src.shape, dtype=src.dtype, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(src); torch.cuda.synchronize(); print("pageable H2D GB/s", round(528e6 / (time.perf_counter() - t) / 1e9, 1))
print("threads default", torch.get_num_threads())
