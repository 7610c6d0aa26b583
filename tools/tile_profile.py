"""Per-tile selection cost of the C2 render (profiling hook gvr_context_set_tile_profile).

Prints the distribution of per-tile select-CTA cycles, the heaviest tiles, the
relation to the tile-list length, and a greedy (LPT) makespan estimate for
148 SMs x the resident CTAs per SM, against the sum of all work. Writes the raw
array to gpurun_out/tile_cycles.npy.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_15401_b200 as gvr  # noqa: E402
from paper_2205_15401_b200 import synthetic  # noqa: E402
from paper_2205_15401_b200.types import SelectionConfig  # noqa: E402


def lpt_makespan(costs, slots):
    import heapq
    h = [0.0] * slots
    for c in sorted(costs, reverse=True):
        t = heapq.heappop(h)
        heapq.heappush(h, t + c)
    return max(h)


def main():
    ctx = gvr.Context()
    ctx.set_tile_profile(True)
    scene = synthetic.make_bench_scene(100000)
    cam = synthetic.make_bench_camera(512)
    ds = gvr.DeviceScene(ctx).set(scene)
    for _ in range(3):
        fr = gvr.render_with_tape(ds, cam, SelectionConfig(), ctx=ctx)
    cyc = fr.tape.tile_cycles().astype(np.float64)
    os.makedirs("gpurun_out", exist_ok=True)
    np.save("gpurun_out/tile_cycles.npy", cyc)
    nz = cyc[cyc > 0]
    print(f"tiles {cyc.size} nonzero {nz.size} sum {nz.sum():.3e} mean {nz.mean():.0f} max {nz.max():.0f}")
    for q in (50, 90, 99, 99.9):
        print(f"  p{q}: {np.percentile(nz, q):.0f}")
    flat = np.argsort(cyc.ravel())[::-1][:20]
    print("top tiles (ty, tx, cycles):", [(int(i // cyc.shape[1]), int(i % cyc.shape[1]), int(cyc.ravel()[i]))
                                          for i in flat])
    for slots in (148, 296, 444):
        ms = lpt_makespan(nz, slots)
        print(f"  LPT makespan over {slots} slots: {ms:.0f} cycles (sum/slots {nz.sum() / slots:.0f})")
    # coarse map, 16x16 blocks of tiles
    ty, tx = cyc.shape
    blk = cyc[: ty // 8 * 8, : tx // 8 * 8].reshape(ty // 8, 8, tx // 8, 8).sum(axis=(1, 3))
    np.set_printoptions(linewidth=200)
    print("coarse map (kcycles per 8x8 tile block):")
    print((blk / 1000).astype(int))


if __name__ == "__main__":
    main()
