"""Numerical probe of the low-rank ("Gram") form of EM-ADMM (development tool, not product).

p_k^t = s p^{t-1} + c^t - a_k lies in span{a_k, c^0..c^t}.  With everything centred on a
per-pixel vector m (translation invariance: the coefficients sum to 0), a sweep needs only
D_k = <a_k - m, c~>, a ring of the last R coefficients of the c~ history per point, and three
scalars per point; the big per-element work is one dot product and one weighted patch sum.

Compares FP32 numpy emulation against the FP64 p-form on seeded NLEM stacks.
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1501_03879_b200 import synth  # noqa: E402


def stacks(img, k, S, pixels):
    hs, hk = S // 2, k // 2
    pad = np.pad(img, hs + hk, mode="reflect")
    H, W = img.shape
    out = []
    for (r, c) in pixels:
        pts = []
        for gy in range(max(0, r - hs), min(H - 1, r + hs) + 1):
            for gx in range(max(0, c - hs), min(W - 1, c + hs) + 1):
                pts.append(pad[gy + hs: gy + hs + k, gx + hs: gx + hs + k].reshape(-1))
        out.append((np.array(pts), pad[r + hs: r + hs + k, c + hs: c + hs + k].reshape(-1)))
    return out


def ref64(A, w, mu, T, box):
    A = A.astype(np.float64)
    w = w.astype(np.float64)
    z = (A * (w / w.sum())[:, None]).sum(0)
    y = np.zeros_like(A)
    lam = w / mu
    n = A.shape[0]
    for _ in range(T):
        v = z - y / mu
        diff = v - A
        nr = np.linalg.norm(diff, axis=1)
        sc = np.where(nr <= lam, 1.0, np.where(nr > 0, lam / np.maximum(nr, 1e-300), 0.0))
        x = v - sc[:, None] * diff
        r = (x + y / mu).sum(0)
        z = np.clip(r / n, *box)
        y = y + mu * (x - z)
    return z


def lr32(A, w, mu, T, box, R, thr_rel=2.0**-22):
    f = np.float32
    A = A.astype(f)
    w = w.astype(f)
    n = A.shape[0]
    z0 = (A * (w / w.sum())[:, None]).sum(0, dtype=f).astype(f)
    m = A[n // 2].copy()  # centre on a patch (any m is exact in real arithmetic)
    At = (A - m).astype(f)
    A2 = (At * At).sum(1, dtype=f)
    lam = (w / f(mu)).astype(f)
    # state (s p = sum_r al[:, r] ch[r] - ga * At): ring of R history vectors
    ch = []  # c~ history (only the live ring)
    al = np.zeros((n, 0), f)
    ga = np.zeros(n, f)
    H = A2.copy()  # ||s p - a~||^2 with s p = 0
    K = -A2.copy()  # <s p - a~, a~>
    z = z0.astype(f)
    zprev = None
    overflow = 0
    for t in range(T):
        c = (z - m) if zprev is None else (f(2) * z - zprev - m)
        c = c.astype(f)
        D = (At @ c).astype(f)
        G = np.array([np.dot(h, c) for h in ch], f)
        Gnn = f(np.dot(c, c))
        X2 = (al @ G).astype(f) if len(ch) else np.zeros(n, f)
        # N = ||s p + c - a||^2 = H + 2<s p - a, c> + ||c||^2
        N = (H + f(2) * (X2 - ga * D - D) + Gnn).astype(f)
        N = np.maximum(N, f(0))
        sc = np.where(lam == 0, f(0), np.minimum(f(1), lam / np.sqrt(N))).astype(f)
        B = (K + D).astype(f)  # <p, a~> = <s p - a~, a~> + <c, a~>
        H = (sc * sc * N - f(2) * sc * B + A2).astype(f)
        K = (sc * B - A2).astype(f)
        ga = (sc * (ga + f(1))).astype(f)
        al = np.concatenate([al * sc[:, None], sc[:, None]], 1).astype(f)
        ch.append(c)
        if len(ch) > R:
            old = np.abs(al[:, 0]) * np.linalg.norm(ch[0])
            if np.any(old > thr_rel * np.sqrt(N)):
                overflow += 1
            al = al[:, 1:]
            ch = ch[1:]
        # g = sum_k s p = sum_r (sum_k al) c~_r - sum_k ga a~_k
        v = al.sum(0, dtype=f)
        g = (sum(v[r] * ch[r] for r in range(len(ch))) - (ga[:, None] * At).sum(0, dtype=f)).astype(f)
        zprev = z
        z = np.clip(z - g / f(n), *box).astype(f)
    return z, overflow


def main():
    rng = np.random.default_rng(0)
    for (size, sig, k, S, T, R) in [(96, 30, 7, 21, 10, 3), (96, 10, 7, 21, 60, 3), (96, 60, 7, 21, 60, 3),
                                    (96, 20, 5, 11, 20, 3), (96, 30, 7, 21, 10, 9)]:
        clean, noisy = synth.noisy_image(size, size, 40, 30, float(sig))
        d = k * k
        h = synth.reference_h(float(sig), d)
        px = [tuple(rng.integers(0, size, 2)) for _ in range(40)] + [(0, 0), (size - 1, 5)]
        worst, ovf = 0.0, 0
        for A, ac in stacks(noisy.astype(np.float64), k, S, px):
            w = np.exp(-((A - ac) ** 2).sum(1) / h ** 2)
            zr = ref64(A, w, 1.0, T, (0, 255))
            zl, o = lr32(A, w, 1.0, T, (0, 255), R)
            worst = max(worst, float(np.abs(zr - zl).max()))
            ovf += o
        print(f"sigma={sig} k={k} S={S} T={T} R={R}: max|z_lr32 - z_ref64| = {worst:.3e}, ring overflows {ovf}")


if __name__ == "__main__":
    main()
