"""Block-buffer slot mapping pinned against the oracle restatement
(oracle/slots.py)."""

import numpy as np
import pytest

from oracle.slots import block_extent, ring_row, storage_row


def test_ring_row_known_answers():
    bs = 3
    assert [ring_row(t, bs) for t in range(12)] == [0, 1, 2, 3, 4, 5, 0, 1, 2, 3, 4, 5]
    assert [storage_row(t, "full") for t in range(4)] == [0, 1, 2, 3]
    assert storage_row(7, "folded") == 0


def test_block_extent_is_the_largest_slice():
    T = 10
    # r[t:min(t+2,T)] over t (nstep2) -> 2; r[t:T] -> T; point access -> 1
    assert block_extent([(t, min(t + 2, T)) for t in range(T)], T) == 2
    assert block_extent([(t, T) for t in range(T)], T) == T
    assert block_extent([], T) == 1


@pytest.mark.parametrize("bs,T", [(2, 6), (3, 6), (4, 10), (5, 5)])
def test_adjust_views_address_equals_ring_row(bs, T):
    """The executor's ring addressing (swap.adjust_views folds -kb*bs*stride
    into the block slot and +(kb mod 2)*bs*stride into the ring slot of
    every view of a managed buffer): the element address of step t, for the
    env values the runtime sets (kb = t // bs, ring = kb mod 2), is the
    oracle's ring row -- bit-exact over every step."""
    from paper_2501_05408_b200 import native as N
    from paper_2501_05408_b200.swap import SwapPlan, adjust_views

    class B:
        pass
    row = 16                      # elements per time step (payload)
    b = B()
    b.ptr, b.dims, b.strides = 1 << 44, ("b", "t"), (2 * bs * row, row)
    v = N.rt_view()
    v.ptr = b.ptr
    slot_t, slot_kb, slot_ring = 0, 1, 2
    v.off_env[slot_t] = row       # the loop over t walks rows of the buffer
    plan = SwapPlan("t", "t_blk", bs, -(-T // bs), slot_ring, [("h", 0)])
    adjust_views([v], plan, {("h", 0): b}, {"t_blk": slot_kb})
    for t in range(T):
        env = {slot_t: t, slot_kb: t // bs, slot_ring: (t // bs) % 2}
        off = v.off + sum(v.off_env[s] * x for s, x in env.items())
        assert off == ring_row(t, bs) * row, (t, off)


@pytest.mark.gpu
@pytest.mark.parametrize("name,bs", [("mlp_f32_I1B4T6", 2), ("mlp_f64_I1B4T6", 3)])
def test_device_ring_rows_hold_the_oracle_slots(name, bs):
    """After a blocked + swapped run the pinned host copy of every managed
    activation -- assembled block by block from device ring rows
    ring_row(t) (written by the acting loop through the adjusted views, read
    by the 2-D offload copies) -- equals the unswapped run's full buffer bit
    for bit, and the device storage is the two-block ring."""
    import torch
    from golden_cases import load_case
    from paper_2501_05408_b200 import execute, executor as X, get_executable
    c = load_case(name)
    X._CACHE.clear()
    ring, _ = get_executable(c.graph(), c.bounds, c.inputs, c.seed, block=("t", bs), swap=1)
    ring.run(c.inputs)
    torch.cuda.synchronize()
    assert ring.swap_plan is not None
    # the same program with the managed activations pinned as outputs: their
    # full (T-step) values, computed by the same acting-loop kernel
    g2 = c.graph()
    keys = list(ring.swap_plan.keys)
    for k in keys:
        g2.outputs.append((f"_pin{k[0]}", k[0], k[1]))
    full = execute(g2, bounds=c.bounds, inputs=c.inputs, seed=c.seed, block=("t", bs))
    for i, k in enumerate(keys):
        rb = ring.bufs[k]
        whole = full[f"_pin{k[0]}"]
        dt = whole.dtype
        host = ring.swap_rt.host[i].numpy().view(dt)[:whole.size].reshape(whole.shape)
        np.testing.assert_array_equal(host, whole, err_msg=str(k))
        # the device storage is the two-block ring (rows ring_row(t) of it)
        ax = rb.dims.index("t")
        T = rb.dshape[ax]
        assert rb.storage_ext()[ax] == 2 * bs
        assert rb.nbytes * T == whole.nbytes * 2 * bs
    X._CACHE.clear()
