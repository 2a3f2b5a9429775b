"""Seeded synthetic workloads for BASELINE.json configs 0-4.

The paper measures on the ONERA M6 and DLR-F6 meshes, which are not
distributed (reference ``SPEC.md:17``). BASELINE.json names synthetic
stand-ins instead; this module builds them exactly as SURVEY.md §8(d)
restates them. Every generator takes a seed, uses ``numpy.random.default_rng``
and returns C-contiguous float64 arrays, (n, 3) AoS, axes x chordwise,
y spanwise, z vertical.

Recorded choices (BASELINE.json leaves them open):

* NACA0012 half-thickness with the closed-trailing-edge coefficient
  a4 = -0.1036 (the same set the reference uses, ``synthetic.py:14``).
* Twist rotates (x - x_qc, z) about the quarter-chord line, nose down for a
  positive angle.
* Config 2's structured grid has 200 span stations x 400 section points,
  u = 2 pi k / 400, xi = (1 + cos u) / 2 (cosine clustering at LE and TE),
  the trailing-edge point appears once. A 1e-9 seeded jitter breaks the
  exact upper/lower mirror symmetry.
* Config 3's fuselage is fixed; its tolerance is 1e-4 * max|d|.
"""

from dataclasses import dataclass

import numpy as np

_A = (0.2969, -0.1260, -0.3516, 0.2843, -0.1036)


def _half_thickness(xi, t_over_c=0.12):
    a0, a1, a2, a3, a4 = _A
    xi = np.clip(xi, 0.0, 1.0)
    return 5.0 * t_over_c * (a0 * np.sqrt(xi) + xi * (a1 + xi * (a2 + xi * (a3 + xi * a4))))


class _SectionArc:
    """Normalised arc length around a unit-chord NACA0012 section.

    u in [0, 2 pi): u = 0 is the trailing edge, the upper surface runs to the
    leading edge at u = pi, the lower surface back to the trailing edge.
    The map s -> u is tabulated once and inverted by interpolation; the
    section scales uniformly with chord, so the table is chord independent.
    """

    def __init__(self, n=200001):
        u = np.linspace(0.0, 2.0 * np.pi, n)
        xi, zc = self.shape(u)
        seg = np.hypot(np.diff(xi), np.diff(zc))
        s = np.concatenate([[0.0], np.cumsum(seg)])
        self.u = u
        self.s = s / s[-1]

    @staticmethod
    def shape(u):
        xi = 0.5 * (1.0 + np.cos(u))
        side = np.where(np.sin(u) >= 0.0, 1.0, -1.0)
        return xi, side * _half_thickness(xi)

    def at(self, s):
        u = np.interp(s, self.s, self.u)
        return self.shape(u)


_ARC = None


def _arc():
    global _ARC
    if _ARC is None:
        _ARC = _SectionArc()
    return _ARC


@dataclass(frozen=True)
class WingGeometry:
    semi_span: float = 1.0
    root_chord: float = 1.0
    tip_chord: float = 0.5
    sweep_deg: float = 25.0
    y0: float = 0.0  # spanwise station of the root

    def chord(self, y):
        frac = (y - self.y0) / (self.semi_span - self.y0)
        return self.root_chord + (self.tip_chord - self.root_chord) * frac

    def x_le(self, y):
        return np.tan(np.radians(self.sweep_deg)) * (y - self.y0)

    def surface(self, y, xi, zc):
        c = self.chord(y)
        return np.column_stack([self.x_le(y) + c * xi, y, c * zc])


def bend_twist(points, geom, bend=0.1, twist_deg=5.0):
    """dz = bend * (y/b)^2 plus a linear twist to ``twist_deg`` at the tip
    about the quarter-chord line (rotation in the x-z plane)."""
    x, y, z = points[:, 0], points[:, 1], points[:, 2]
    eta = y / geom.semi_span
    theta = np.radians(twist_deg) * eta
    x_qc = geom.x_le(y) + 0.25 * geom.chord(y)
    rx = x - x_qc
    c, s = np.cos(theta), np.sin(theta)
    dx = rx * (c - 1.0) + z * s
    dz = -rx * s + z * (c - 1.0) + bend * eta * eta
    return np.ascontiguousarray(np.column_stack([dx, np.zeros_like(dx), dz]))


def volume_cloud(rng, surface, nv, mean_exp=0.05, spread=2.0):
    """Volume nodes v = p_k + delta * u, k ~ U{0..Nb-1}, u uniform on the
    sphere, delta ~ Exp(mean_exp) + U(0, spread)."""
    k = rng.integers(0, len(surface), nv)
    u = rng.normal(size=(nv, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    delta = rng.exponential(mean_exp, nv) + rng.uniform(0.0, spread, nv)
    return np.ascontiguousarray(surface[k] + delta[:, None] * u)


@dataclass
class Workload:
    name: str
    points: np.ndarray  # boundary (Nb, 3)
    disp: np.ndarray  # prescribed (Nb, 3)
    volume: np.ndarray  # (Nv, 3)
    radius: float
    tol: float
    m: int
    seed: int = 0

    @property
    def nb(self):
        return len(self.points)

    @property
    def nv(self):
        return len(self.volume)


def _tol(disp, frac):
    return float(frac * np.linalg.norm(disp, axis=1).max())


def random_wing(nb, nv, seed=0, m=8, radius=2.0, tol_frac=1e-4, name="cfg0"):
    """Configs 0 and 1: (y, s) iid U[0, b] x U[0, 1] on the tapered wing."""
    rng = np.random.default_rng(seed)
    geom = WingGeometry()
    y = rng.uniform(0.0, geom.semi_span, nb)
    s = rng.uniform(0.0, 1.0, nb)
    xi, zc = _arc().at(s)
    pts = np.ascontiguousarray(geom.surface(y, xi, zc))
    disp = bend_twist(pts, geom)
    vol = volume_cloud(rng, pts, nv)
    return Workload(name, pts, disp, vol, radius, _tol(disp, tol_frac), m, seed)


def structured_wing(n_span=200, n_section=400, nv=10_000_000, seed=0, m=48,
                    radius=2.0, tol_frac=1e-5, name="cfg2"):
    """Config 2: span x arc structured grid with cosine LE/TE clustering."""
    rng = np.random.default_rng(seed)
    geom = WingGeometry()
    y = np.linspace(0.0, geom.semi_span, n_span)
    u = 2.0 * np.pi * np.arange(n_section) / n_section
    xi, zc = _SectionArc.shape(u)
    yy = np.repeat(y, n_section)
    pts = geom.surface(yy, np.tile(xi, n_span), np.tile(zc, n_span))
    pts = np.ascontiguousarray(pts + 1e-9 * rng.uniform(-1.0, 1.0, pts.shape))
    disp = bend_twist(pts, geom)
    vol = volume_cloud(rng, pts, nv)
    return Workload(name, pts, disp, vol, radius, _tol(disp, tol_frac), m, seed)


def wing_body(nb=200_000, nv=40_000_000, seed=0, m=64, radius=4.0, tol_frac=1e-4,
              name="cfg3"):
    """Config 3: fuselage + wing + pylon + nacelle, points split by area.

    Fuselage: cylinder r = 0.4 over x in [0, 6] with an ogive (tangent
    circular-arc) nose over the first 1.2, fixed (zero displacement).
    Wing: the config-0 wing scaled uniformly by 3 (semi-span 3, chord
    3.0 -> 1.5, 25 deg sweep, NACA0012), leading edge at x = 2 on the
    centre line; only its exposed part, y in [0.4, 3] (outboard of the
    fuselage radius), carries points. Pylon: a flat plate of height 0.25 at
    y = 1.2, hung below the wing's thickest point (z <= -0.15). Nacelle:
    cylindrical shell r = 0.15, length 0.8, below the pylon. Pylon and
    nacelle move rigidly with the wing section at y = 1.2.
    """
    rng = np.random.default_rng(seed)
    b = 3.0
    geom = WingGeometry(semi_span=b, root_chord=3.0, tip_chord=1.5)
    y_root = 0.4  # fuselage radius: the wing is exposed over y in [0.4, 3]
    x_root = 2.0
    r_f, l_f, l_nose = 0.4, 6.0, 1.2
    y_p, r_n, l_n = 1.2, 0.15, 0.8

    # component areas (approximate, for the point split)
    a_fus = 2 * np.pi * r_f * (l_f - l_nose) + np.pi * r_f * np.hypot(r_f, l_nose)
    span_w = b - y_root
    a_wing = 2.04 * 0.5 * (geom.chord(y_root) + geom.tip_chord) * span_w
    c_p = geom.chord(y_p)
    h_p = 0.25
    z_p = 0.15  # below the wing's half-thickness at y_p (0.06 * chord = 0.144)
    a_pyl = 2 * 0.6 * c_p * h_p
    a_nac = 2 * np.pi * r_n * l_n
    areas = np.array([a_fus, a_wing, a_pyl, a_nac])
    counts = np.floor(nb * areas / areas.sum()).astype(int)
    counts[1] += nb - counts.sum()

    def fuselage(n):
        # area-weighted sampling along x: cylinder plus ogive nose
        x = np.empty(0)
        while len(x) < n:
            cand = rng.uniform(0.0, l_f, 2 * n)
            r = np.where(cand < l_nose, r_f * np.sqrt(np.clip(cand / l_nose * (2 - cand / l_nose), 0, 1)), r_f)
            keep = rng.uniform(0.0, r_f, len(cand)) < r
            x = np.concatenate([x, cand[keep]])
        x = x[:n]
        r = np.where(x < l_nose, r_f * np.sqrt(np.clip(x / l_nose * (2 - x / l_nose), 0, 1)), r_f)
        ang = rng.uniform(0.0, 2 * np.pi, n)
        return np.column_stack([x, r * np.cos(ang), r * np.sin(ang)])

    def wing(n):
        y = rng.uniform(y_root, b, n)
        s = rng.uniform(0.0, 1.0, n)
        xi, zc = _arc().at(s)
        p = geom.surface(y, xi, zc)
        p[:, 0] += x_root
        return p

    x_le_p = x_root + geom.x_le(y_p)

    def pylon(n):
        xs = x_le_p + c_p * rng.uniform(0.2, 0.8, n)
        zs = -rng.uniform(0.0, h_p, n) - z_p
        side = np.where(rng.uniform(size=n) < 0.5, -0.005, 0.005)
        return np.column_stack([xs, y_p + side, zs])

    def nacelle(n):
        xs = x_le_p - 0.3 + rng.uniform(0.0, l_n, n)
        ang = rng.uniform(0.0, 2 * np.pi, n)
        zc = -z_p - h_p - r_n - 0.02
        return np.column_stack([xs, y_p + r_n * np.cos(ang), zc + r_n * np.sin(ang)])

    parts = [fuselage(counts[0]), wing(counts[1]), pylon(counts[2]), nacelle(counts[3])]
    pts = np.ascontiguousarray(np.concatenate(parts))
    disp = np.zeros_like(pts)
    nf, nw, npyl = counts[0], counts[1], counts[2]
    wing_pts = pts[nf:nf + nw].copy()
    wing_pts[:, 0] -= x_root
    wgeom = geom
    disp[nf:nf + nw] = bend_twist(wing_pts, wgeom, bend=0.2, twist_deg=3.0)
    # rigid motion of pylon + nacelle with the wing section at y_p
    eng = pts[nf + nw:].copy()
    eng_local = eng.copy()
    eng_local[:, 0] -= x_root
    eng_local[:, 1] = y_p
    disp[nf + nw:] = bend_twist(eng_local, wgeom, bend=0.2, twist_deg=3.0)
    vol = volume_cloud(rng, pts, nv)
    return Workload(name, pts, disp, vol, radius, _tol(disp, tol_frac), m, seed)


def config(idx, seed=0, nv=None):
    """Workload for BASELINE.json ``configs[idx]`` (idx 0-3)."""
    if idx == 0:
        return random_wing(2000, nv or 100_000, seed=seed, m=8, name="cfg0")
    if idx == 1:
        return random_wing(20_000, nv or 2_000_000, seed=seed, m=32, name="cfg1")
    if idx == 2:
        return structured_wing(nv=nv or 10_000_000, seed=seed)
    if idx == 3:
        return wing_body(nv=nv or 40_000_000, seed=seed)
    raise ValueError(f"unknown config {idx}")
