"""The SPEC's runtime Backend + MemorySim over the C ABI (csrc/backend.cu).

Reference SPEC.md:541-561: `Backend — allocate, deallocate,
move-between-tiers, execute-kernel(kind, inputs, params), dynamic-update,
stack` and `MemorySim — device tier {capacity, live, peak}; host tier
{live, peak}; transfer counters {fetches, offloads, bytes moved}; device
overflow is a hard error`.  The reference package specifies these and
implements none of them.  Here:

    allocate / deallocate   stream-ordered pool (cudaMallocFromPoolAsync)
    move_between_tiers      offload / fetch: pinned 2-D copies on a copy
                            stream, ordered by and recording CUDA events
    execute_kernel          rt_launch (one kernel family, KERNELS-table ABI)
    dynamic_update          one point's value into a block slot (BlockStore)
    stack                   point values concatenated (slice materialised)
    stats()                 the MemorySim counters

The executor's swapping (swap.py) moves its time blocks through this API.
"""

from __future__ import annotations

import ctypes as C

from . import native as N


class OverflowError_(Exception):
    """MemorySim: device overflow is a hard error."""


STAT_KEYS = ("capacity", "live", "peak", "host_live", "host_peak", "offloads", "fetches",
             "bytes_moved")


class Backend:
    def __init__(self, device: int = 0, capacity: int = 0):
        self.lib = N.lib()
        h = N.u64()
        N.check(self.lib.rt_pool_create(int(device), int(capacity), C.byref(h)), "pool create")
        self.pool = h.value

    def close(self):
        if self.pool:
            N.check(self.lib.rt_pool_destroy(self.pool), "pool destroy")
            self.pool = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # allocate / deallocate ---------------------------------------------------
    def allocate(self, nbytes: int, stream: int = 0) -> int:
        out = N.u64()
        rc = self.lib.rt_pool_alloc(self.pool, int(nbytes), int(stream), C.byref(out))
        if rc == N.RT_ERR_OVERFLOW:
            raise OverflowError_(self.lib.rt_last_error().decode())
        N.check(rc, "allocate")
        return out.value

    def deallocate(self, ptr: int, stream: int = 0):
        N.check(self.lib.rt_pool_free(self.pool, int(ptr), int(stream)), "deallocate")

    # move-between-tiers ----------------------------------------------------
    def offload(self, host_ptr: int, dev_ptr: int, width: int, height: int = 1, hpitch: int = 0,
                dpitch: int = 0, stream: int = 0, after_event: int = 0, done_event: int = 0):
        N.check(self.lib.rt_offload(self.pool, C.c_void_p(host_ptr), int(hpitch or width),
                                    int(dev_ptr), int(dpitch or width), int(width), int(height),
                                    int(stream), int(after_event), int(done_event)), "offload")

    def fetch(self, dev_ptr: int, host_ptr: int, width: int, height: int = 1, dpitch: int = 0,
              hpitch: int = 0, stream: int = 0, after_event: int = 0, done_event: int = 0):
        N.check(self.lib.rt_fetch(self.pool, int(dev_ptr), int(dpitch or width),
                                  C.c_void_p(host_ptr), int(hpitch or width), int(width),
                                  int(height), int(stream), int(after_event), int(done_event)),
                "fetch")

    def host_tier(self, delta_bytes: int):
        N.check(self.lib.rt_pool_host(self.pool, int(delta_bytes)), "host tier")

    # execute-kernel ----------------------------------------------------------
    def execute_kernel(self, rec, env=(), stream: int = 0):
        arr = (N.i64 * max(1, len(env)))(*env)
        N.check(self.lib.rt_launch(C.byref(rec), arr, len(env), int(stream)), "execute kernel")

    # dynamic-update / stack --------------------------------------------------
    def dynamic_update(self, block_ptr: int, slot: int, src_ptr: int, elem_bytes: int,
                       stream: int = 0):
        N.check(self.lib.rt_block_update(int(block_ptr), int(slot), int(src_ptr),
                                         int(elem_bytes), int(stream)), "dynamic update")

    def stack(self, dst_ptr: int, src_ptrs, elem_bytes: int, stream: int = 0):
        arr = (N.u64 * max(1, len(src_ptrs)))(*[int(p) for p in src_ptrs])
        N.check(self.lib.rt_stack(int(dst_ptr), arr, len(src_ptrs), int(elem_bytes), int(stream)),
                "stack")

    # MemorySim -----------------------------------------------------------------
    def stats(self) -> dict:
        v = (N.u64 * 8)()
        N.check(self.lib.rt_pool_stats(self.pool, v), "stats")
        return dict(zip(STAT_KEYS, (int(x) for x in v)))
