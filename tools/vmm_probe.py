"""Host cost of CUDA VMM operations (the pooled expert memory's per-load work), GPU box.

    python tools/vmm_probe.py
Maps / unmaps 2 GiB (one C5 8192 x 61440 expert) as pages of 2 / 8 / 32 / 128 MB and prints
the host time per expert for cuMemMap + cuMemSetAccess and for cuMemUnmap.
"""
import time

from cuda.bindings import driver as cu


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(err)
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


ck(cu.cuInit(0))
dev = ck(cu.cuDeviceGet(0))
ctx = ck(cu.cuDevicePrimaryCtxRetain(dev))
ck(cu.cuCtxSetCurrent(ctx))
prop = cu.CUmemAllocationProp()
prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
prop.location.id = 0
acc = cu.CUmemAccessDesc()
acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
acc.location.id = 0
acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
total = 2 << 30
for page_mb in (2, 8, 32, 128):
    page = page_mb << 20
    n = total // page
    hs = [ck(cu.cuMemCreate(page, prop, 0)) for _ in range(n)]
    va = ck(cu.cuMemAddressReserve(total, page, 0, 0))
    t_map = t_unmap = 0.0
    reps = 5
    for _ in range(reps):
        t0 = time.perf_counter()
        for i, h in enumerate(hs):
            ck(cu.cuMemMap(int(va) + i * page, page, 0, h, 0))
        ck(cu.cuMemSetAccess(va, total, [acc], 1))
        t1 = time.perf_counter()
        for i in range(n):
            ck(cu.cuMemUnmap(int(va) + i * page, page))
        t2 = time.perf_counter()
        t_map += t1 - t0
        t_unmap += t2 - t1
    print(f"page {page_mb:4d} MB x {n:5d}: map+access {1e3 * t_map / reps:8.2f} ms, unmap {1e3 * t_unmap / reps:8.2f} ms "
          f"per 2 GiB expert", flush=True)
    ck(cu.cuMemAddressFree(va, total))
    for h in hs:
        ck(cu.cuMemRelease(h))
