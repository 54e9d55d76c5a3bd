"""Shared-memory bank-conflict model of the tiled walk's position gathers on
realistic lists (uniform rho = 0.75 box, CSF-1 grid, z-sorted cells, the
walk's 2 x 2 x TZ tiles and 4 x 4-column windows, inner lists at rp = 2.6).

Compares, per 8-byte LDS of a warp (two half-warp wavefront groups):
  (a) lane = row, entries in ascending window order (the walk as built);
  (b) half-warp = row, the row's entries sorted by bank (window index mod 16)
      and dealt over T = ceil(n / 16) steps: lane l takes sorted entries
      [l*T, l*T + T), so step t holds entries l*T + t.
Wavefronts of one half-warp access = the largest number of distinct window
rows falling into one bank.

    python tools/experiments/bank_sim.py [--n 200000]
"""
import argparse

import numpy as np
from scipy.spatial import cKDTree


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--rp", type=float, default=2.6)
    ap.add_argument("--tz", type=int, default=4)
    ap.add_argument("--extra", type=int, default=0)
    ap.add_argument("--adaptive", action="store_true")
    ap.add_argument("--two-choice", type=int, default=0,
                    help="(a) with every window row stored twice, the copy offset by this many banks; "
                         "each half-warp access picks a copy greedily (lane order)")
    ap.add_argument("--consecutive", action="store_true",
                    help="(c): no bank sort, step t = ascending entries [16t, 16t+16)")
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    L = (a.n / 0.75) ** (1 / 3)
    pos = rng.random((a.n, 3)) * L
    S = int(L // 2.8)
    cl = L / S
    c = np.minimum((pos // cl).astype(int), S - 1)
    flat = (c[:, 0] * S + c[:, 1]) * S + c[:, 2]
    order = np.lexsort((pos[:, 2], flat))
    pos, c, flat = pos[order], c[order], flat[order]
    start = np.searchsorted(flat, np.arange(S ** 3 + 1))
    tree = cKDTree(pos, boxsize=L)
    tz = a.tz
    res_a, res_b, slots_a, slots_b, ent = [], [], 0, 0, 0
    ntile = 0
    for x0 in range(1, S - 3, 2):
        for y0 in range(1, S - 3, 2):
            for z0 in range(1, S - tz - 1, tz):
                ntile += 1
                if ntile > 60:
                    break
                za, zb = z0 - 1, z0 + tz
                widx = {}
                off = 0
                for aa in range(4):
                    for bb in range(4):
                        col = (x0 - 1 + aa) * S + (y0 - 1 + bb)
                        ws = start[col * S + za] & ~3
                        we = (start[col * S + zb + 1] + 3) & ~3
                        for r in range(start[col * S + za], start[col * S + zb + 1]):
                            widx[r] = off + (r - ws)
                        off += we - ws
                rows = []
                for aa in range(2):
                    for bb in range(2):
                        col = (x0 + aa) * S + (y0 + bb)
                        rows.extend(range(start[col * S + z0], start[col * S + z0 + tz]))
                lists = []
                for r in rows:
                    nb = tree.query_ball_point(pos[r], a.rp)
                    w = sorted(widx[j] for j in nb if j != r)
                    lists.append(np.array(w, dtype=np.int64))
                # (a) lane per row, ascending window order
                for q0 in range(0, len(lists), 32):
                    chunk = lists[q0:q0 + 32]
                    kmax = max(len(x) for x in chunk)
                    slots_a += 32 * kmax
                    for k in range(kmax):
                        wf = 0
                        for h in (chunk[:16], chunk[16:]):
                            addr = sorted({x[k] for x in h if k < len(x)})
                            if addr and a.two_choice:
                                load = np.zeros(16, dtype=int)
                                for ad in addr:
                                    b0, b1 = ad % 16, (ad + a.two_choice) % 16
                                    load[b0 if load[b0] <= load[b1] else b1] += 1
                                wf += load.max()
                            elif addr:
                                banks = np.bincount(np.array(addr) % 16, minlength=16)
                                wf += banks.max()
                        res_a.append(wf)
                # (b) half-warp per row, bank-sorted and dealt
                for i in range(0, len(lists), 2):
                    pair = lists[i:i + 2]
                    steps = []
                    for w in pair:
                        n = len(w)
                        ent += n
                        T = max(1, -(-n // 16)) + a.extra
                        if a.adaptive:
                            cb = np.bincount(w % 16, minlength=16).max()
                            if cb > T and -(-cb // T) > -(-cb // (T + 1)):
                                T += 1
                        srt = w[np.lexsort((w, w % 16))]
                        st = []
                        for t in range(T):
                            if a.consecutive:
                                st.append(w[16 * t:16 * t + 16])
                                continue
                            e = np.arange(16) * T + t
                            st.append(srt[e[e < n]])
                        steps.append(st)
                    tmax = max(len(s) for s in steps)
                    slots_b += 32 * tmax
                    for t in range(tmax):
                        wf = 0
                        for st in steps:
                            if t < len(st) and len(st[t]):
                                addr = np.unique(st[t])
                                wf += np.bincount(addr % 16, minlength=16).max()
                        res_b.append(wf)
    ra, rb = np.array(res_a), np.array(res_b)
    # cost model per warp step: 18 FP64 warp instructions = 9 SM-clk; shared:
    # 3 gathers x wavefronts + 1 list wavefront (1 wavefront / clk / SM)
    for nm, r in (("a", ra), ("b", rb)):
        fp, sh = 9 * len(r), 3 * r.sum() + len(r)
        print(f"  model {nm}: fp64 {fp / ent:.3f} clk/entry  shared {sh / ent:.3f} clk/entry  bound {max(fp, sh) / ent:.3f}")
    print(f"tiles {min(ntile, 60)}  entries {ent}")
    print(f"(a) lane/row : wavefronts per warp LDS {ra.mean():.2f} (ideal 2)  "
          f"LDS per entry {len(ra) / ent:.4f}  wavefronts per entry {ra.sum() / ent:.3f}  "
          f"slot eff {ent / slots_a:.3f}")
    print(f"(b) halfwarp : wavefronts per warp LDS {rb.mean():.2f} (ideal 2)  "
          f"LDS per entry {len(rb) / ent:.4f}  wavefronts per entry {rb.sum() / ent:.3f}  "
          f"slot eff {ent / slots_b:.3f}")


if __name__ == "__main__":
    main()
