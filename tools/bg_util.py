"""Print the lane-utilisation model (gen/lower_bg.py lane_utilisation) of the Berends-Giele plans:
the default plan of each size and every subset-batch candidate, with shared memory and occupancy.
usage: python tools/bg_util.py [N ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2511_19456_b200.gen.emit import choose_launch  # noqa: E402
from paper_2511_19456_b200.gen.lower_bg import lane_utilisation, make_bg_plan  # noqa: E402


def show(p, tag):
    util, by = lane_utilisation(p)
    span = sum(a[0] for a in by.values())
    wpb, blocks = choose_launch(p)
    parts = "  ".join(f"{k} {100 * a[0] / span:4.1f}%/{a[1] / (p.G * a[0]):.2f}" for k, a in by.items())
    print(f"{tag} N={p.N} setb={p.setb} store={p.store} smem/pt={p.stride * 8 / 1024:6.1f} KB "
          f"warps/SM={wpb * blocks:2d} util={util:.3f}  [{parts}]")


if __name__ == "__main__":
    for N in (map(int, sys.argv[1:]) if len(sys.argv) > 1 else range(2, 10)):
        d = make_bg_plan(N)
        show(d, "default")
        for b in (1, 2, 4, 8):
            if b != d.setb and b <= len(d.sets):
                try:
                    show(make_bg_plan(N, setb=b), "      ")
                except Exception as e:  # noqa: BLE001
                    print("      ", N, b, e)
