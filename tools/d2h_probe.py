import mmap, time
import numpy as np, torch
x = torch.randn(128, 257, 257, dtype=torch.complex128, device="cuda")
nb = x.numel() * 16
stage = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
def t(label, fn, n=4):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): r = fn()
    torch.cuda.synchronize(); print(f"{label}: {(time.perf_counter()-t0)/n*1e3:.1f} ms", flush=True)
t("x.cpu().numpy()", lambda: x.cpu().numpy())
def staged_copy():
    stage.copy_(x); a = np.empty(x.shape, np.complex128); np.copyto(a, stage.numpy()); return a
t("pinned stage + np.copyto", staged_copy)
def thp():
    m = mmap.mmap(-1, nb, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(m, dtype=np.complex128).reshape(x.shape)
    torch.from_numpy(a).copy_(x); return a
t("THP buffer, pageable D2H", thp)
def thp_staged():
    m = mmap.mmap(-1, nb, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(m, dtype=np.complex128).reshape(x.shape)
    stage.copy_(x); np.copyto(a, stage.numpy()); return a
t("THP buffer, pinned stage + copyto", thp_staged)
t("pinned stage only", lambda: stage.copy_(x))
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
