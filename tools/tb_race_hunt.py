"""Find the first two-step launch whose result differs from two one-step
steps (debugging tool).

python tools/tb_race_hunt.py [lx ly launches trials l2]

Two lattices from the same RT state: the reference on the one-step kernel
and the subject on the two-step kernel (TMA L2 prefetch distance l2).  After
every launch (2 steps) both are synchronised and their current buffers
compared on the device; at the first difference the differing entries are
decoded from the internal layout ((ix * 37 + l) * nyp + r) into
(population, physical column, physical row) and printed with the strip and
the CTA column ranges that wrote them.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lbgen  # noqa: E402
import paper_1703_00186_b200 as lbm  # noqa: E402


def main():
    a = [int(v) for v in sys.argv[1:6]]
    lx, ly, launches, trials, l2 = a if len(a) == 5 else (1920, 2048, 500, 8, 4)
    T0 = 1.0 / 1.19697977039307435897239 ** 2
    found = []
    for trial in range(trials):
        sr, st = torch.cuda.Stream(), torch.cuda.Stream()
        ref = lbm.Lattice(lx, ly, stream=sr, temporal=False)
        sub = lbm.Lattice(lx, ly, stream=st, temporal=False)
        sub.temporal(True, l2_prefetch=l2)
        for g in (ref, sub):
            g.init_macro(*lbgen.rt_macro(lx, ly, T0))
            g.step(20)
            g.sync()
        L = ref.layout
        nyp, y0 = int(L.nyp), int(L.y0)

        def phys(t):
            return t.view(-1, 37, nyp)[3:3 + lx, :, y0:y0 + ly]

        # the one-step path swaps its buffers every step, the two-step path
        # once per launch: find which buffers hold the state now, then follow
        def current(g):  # index of the buffer lb_peek_cols(which = 0) reads
            c0 = torch.from_numpy(g.peek_cols(0, 1)[:, 0, :]).to(g.bufs[0].device)
            return 0 if torch.equal(phys(g.bufs[0])[0], c0) else 1

        ia, ib = current(ref), current(sub)
        assert torch.equal(phys(ref.bufs[ia]), phys(sub.bufs[ib])), "states differ after the warm-up"
        bad = None
        for k in range(launches):
            ref.step(2)
            ref.sync()
            sub.step(2)
            sub.sync()
            ib ^= 1
            x, y = phys(ref.bufs[ia]), phys(sub.bufs[ib])
            if not torch.equal(x, y):
                d = torch.nonzero(x != y)  # (column, population, row)
                pts = [[int(v[1]), int(v[0]), int(v[2])] for v in d[:12]]
                bad = {"trial": trial, "launch": k, "n_diff": int(len(d)), "first_pop_col_row": pts,
                       "rows": sorted(set(int(v) for v in d[:4096, 2]))[:40],
                       "cols": sorted(set(int(v) for v in d[:4096, 0]))[:40],
                       "pops": sorted(set(int(v) for v in d[:4096, 1]))}
                break
        rec = bad or {"trial": trial, "launch": launches, "n_diff": 0}
        print(json.dumps(rec), flush=True)
        if bad:
            found.append(bad)
        ref.close()
        sub.close()
        del ref, sub
        torch.cuda.empty_cache()
    print(json.dumps({"trials": trials, "launches_each": launches, "found": len(found)}))


if __name__ == "__main__":
    main()
