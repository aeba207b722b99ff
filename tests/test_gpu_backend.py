"""The SPEC runtime Backend + MemorySim at the C ABI (csrc/backend.cu,
backend.py; reference SPEC.md:541-561): allocate / deallocate with live and
peak accounting and the overflow hard error, tier moves ordered by events,
dynamic-update into a block slot, stack of point values."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_pool_accounting_and_overflow():
    from paper_2501_05408_b200.backend import Backend, OverflowError_
    be = Backend(0, capacity=1 << 20)
    a = be.allocate(600_000)
    b = be.allocate(300_000)
    st = be.stats()
    assert st["live"] == 900_000 and st["peak"] == 900_000 and st["capacity"] == 1 << 20
    with pytest.raises(OverflowError_):
        be.allocate(200_000)
    be.deallocate(a)
    c = be.allocate(200_000)
    st = be.stats()
    assert st["live"] == 500_000 and st["peak"] == 900_000
    be.deallocate(b)
    be.deallocate(c)
    assert be.stats()["live"] == 0
    be.close()


def test_tier_moves_block_update_and_stack():
    import torch
    from paper_2501_05408_b200.backend import Backend
    be = Backend(0)
    s = torch.cuda.Stream()
    x = np.arange(4 * 1000, dtype=np.float32).reshape(4, 1000)
    host = torch.from_numpy(x.copy()).pin_memory()
    back = torch.zeros_like(host).pin_memory()
    dev = be.allocate(x.nbytes, s.cuda_stream)
    ev_in, ev_out = torch.cuda.Event(), torch.cuda.Event()
    # fetch rows 0 and 2 (a 2-D move: 2 rows of 4 KB, host pitch 8 KB)
    be.fetch(dev, host.data_ptr(), 4000, 2, dpitch=4000, hpitch=8000, stream=s.cuda_stream,
             done_event=ev_in.cuda_event)
    be.offload(back.data_ptr(), dev, 8000, stream=s.cuda_stream, after_event=ev_in.cuda_event,
               done_event=ev_out.cuda_event)
    ev_out.synchronize()
    got = back.numpy()
    assert np.array_equal(got[0], x[0]) and np.array_equal(got[1], x[2])
    st = be.stats()
    assert st["fetches"] == 1 and st["offloads"] == 1 and st["bytes_moved"] == 16000
    # dynamic-update: point values into slots of a pre-allocated block
    blk = torch.zeros(6, 16, dtype=torch.float64, device="cuda")
    pts = [torch.full((16,), float(i + 1), dtype=torch.float64, device="cuda") for i in range(3)]
    cur = torch.cuda.current_stream().cuda_stream
    for slot, p in zip((4, 0, 2), pts):
        be.dynamic_update(blk.data_ptr(), slot, p.data_ptr(), 16 * 8, cur)
    want = np.zeros((6, 16))
    want[4], want[0], want[2] = 1, 2, 3
    assert np.array_equal(blk.cpu().numpy(), want)
    # stack: 300 points (two kernel batches), odd element size (no vectors)
    srcs = [torch.arange(i, i + 13, dtype=torch.uint8, device="cuda") for i in range(300)]
    dst = torch.empty(300 * 13, dtype=torch.uint8, device="cuda")
    be.stack(dst.data_ptr(), [t.data_ptr() for t in srcs], 13, cur)
    assert np.array_equal(dst.cpu().numpy().reshape(300, 13),
                          np.stack([t.cpu().numpy() for t in srcs]))
    be.deallocate(dev, s.cuda_stream)
    torch.cuda.synchronize()
    be.close()


def test_swapped_run_moves_blocks_through_the_backend():
    """swap.py's offload/fetch go through the Backend: its MemorySim counts
    one offload and one fetch per swapped buffer per time block."""
    from golden_cases import load_case
    from paper_2501_05408_b200 import get_executable
    c = load_case("mlp_f32_I1B4T6")
    exe, _ = get_executable(c.graph(), c.bounds, c.inputs, c.seed, block=("t", 2), swap=1)
    exe.run(c.inputs)
    exe.fetch()
    st = exe.swap_rt.backend.stats()
    keys, blocks = len(exe.swap_plan.keys), exe.swap_plan.DI
    assert st["offloads"] == keys * blocks and st["fetches"] == keys * blocks
    assert st["host_live"] == exe.swap_rt.host_bytes and st["bytes_moved"] > 0
