"""Summarise a QT_MK_TRACE dump of the persistent decode kernel: per phase, the
span from the earliest CTA entering to the last CTA leaving, and the median
per-CTA duration, averaged over layers 1..L-2."""
import sys
import numpy as np

NAMES = ["S0 owner norm+quant / wait", "S1 QKV GEMV", "S1 barrier", "S2 attention units", "S2 wait attn rows",
         "S4 O GEMV", "S4 barrier", "S5 owner+wait", "S6 GU GEMV", "S6 barrier", "S7 owner+wait", "S8 down GEMV",
         "S8 barrier"]


def main(path, G, L):
    t = np.fromfile(path, dtype=np.uint64).astype(np.float64).reshape(G, L + 1, 32)
    t0 = t[:, :L, 0].min()
    print(f"step span {(t[:, L, 3].max() - t[:, 0, 0].min()) / 1e3:.1f} us (layer-0 start -> head barrier)")
    tot = 0
    for k in range(1, 14):
        d = (t[:, 1:L - 1, k] - t[:, 1:L - 1, k - 1]) / 1e3  # us, per CTA per layer
        med = np.median(d)
        mx = d.max(axis=0).mean()
        tot += np.median(d.mean(axis=1))
        print(f"{NAMES[k - 1]:30s} median {med:7.2f} us   mean-of-max {mx:7.2f} us")
    lay = (t[:, 2:L - 1, 0] - t[:, 1:L - 2, 0]) / 1e3
    print(f"per layer: {np.median(lay):.2f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))


def owners(path, G, L, B=8):
    t = np.fromfile(path, dtype=np.uint64).astype(np.float64).reshape(G, L + 1, 32)
    d0 = (t[:B, 1:L - 1, 14] - t[:B, 1:L - 1, 0]) / 1e3
    d7 = (t[:B, 1:L - 1, 15] - t[:B, 1:L - 1, 10]) / 1e3
    print(f"owner S0 work {np.median(d0):.2f} us, owner S7 work {np.median(d7):.2f} us")
    sub = [(t[:B, 1:L - 1, k] - t[:B, 1:L - 1, j]) / 1e3 for j, k in ((0, 16), (16, 17), (17, 18), (18, 19), (19, 20))]
    print("S0 owner: loop1 %.2f  wk_sum %.2f  loop2 %.2f  max %.2f  quant %.2f us" % tuple(np.median(x) for x in sub))


if len(sys.argv) > 4:
    owners(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
