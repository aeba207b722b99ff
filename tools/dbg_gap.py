import sys, numpy as np
sys.path[:0] = [".", "tests"]
from test_swap_gap import gap_graph
from paper_2501_05408_b200 import executor as X, get_executable, memplan, swap as SW
import paper_2501_05408_b200.swap as SWM
orig = SWM.plan_gap_swap
def wrapped(prog, rec_ptrs, key_of, managed, sizes, base_life, assign, lifetimes_of):
    print("managed", managed)
    t = SWM.key_touches(prog, rec_ptrs, key_of)
    for k in managed: print(" touches", k, t.get(k), SWM._segments(prog, t.get(k, ())))
    print("cands", SWM.gap_candidates(prog, t, managed))
    print("base arena", assign(sizes, base_life)[1])
    for pc, ins in enumerate(prog): print("  pc", pc, ins[:2], [key_of.get(p) for p in (rec_ptrs[ins[1]] if ins[0]==1 else ())])
    r = orig(prog, rec_ptrs, key_of, managed, sizes, base_life, assign, lifetimes_of)
    print("chosen", r[0])
    return r
SWM.plan_gap_swap = wrapped
B, T, H = 64, 256, 256
rng = np.random.default_rng(0)
x = rng.standard_normal((B, T, 1, H)).astype(np.float32)
W = (rng.standard_normal((H, H)) / 16).astype(np.float32)
g = gap_graph(B, T, H)
exe, _ = get_executable(g, {}, {"x": x, "W": W}, 0, swap=1 << 20)
print("labels", exe.labels)
print("names", exe.trace_names)
