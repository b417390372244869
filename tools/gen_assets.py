"""Generates the synthetic hand specs and mesh object the benchmark configs
name (BASELINE.json configs; SURVEY.md 7 "Hand specs to author").

The reference ships only the 3-finger trident (proj/src/hand.cpp:365-453);
Allegro, Leap and Shadow are MuJoCo assets the SPEC excludes.
These are stand-ins in the reference's own hand-spec format
(proj/src/hand.cpp:259-363): one revolute joint per link, >= 4
non-coplanar vertices per link, tiny "knuckle" links for multi-DoF joints,
fingers along +z from the palm like the trident, flexion curling toward the
opposing digit. Both the oracle and the GPU engine consume the same spec.

    python tools/gen_assets.py   # writes paper_2412_16490_b200/assets/
"""
from __future__ import annotations

import json
import math
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "paper_2412_16490_b200" / "assets"


def box(cx, cy, z0, z1, hx, hy):
    return [[cx + sx * hx, cy + sy * hy, z] for sx in (-1, 1) for sy in (-1, 1) for z in (z0, z1)]


def tip_shell(center, radius, n=48):
    golden = math.pi * (3.0 - math.sqrt(5.0))
    pts = []
    for k in range(n):
        z = 1.0 - 2.0 * (k + 0.5) / n
        r = math.sqrt(max(1.0 - z * z, 0.0))
        pts.append([center[0] + radius * r * math.cos(golden * k), center[1] + radius * r * math.sin(golden * k),
                    center[2] + radius * z])
    return pts


def r6(v):
    return [round(float(c), 6) for c in v]


class Spec:
    def __init__(self, name):
        self.doc = {"format_version": 1, "name": name, "links": [], "ignore_collisions": []}
        self.fingers = {}

    def link(self, name, verts, proxies=(), joint=None, tip=None):
        d = {"name": name, "vertices": [r6(v) for v in verts]}
        if proxies:
            d["proxies"] = [{"center": r6(c), "radius": r} for c, r in proxies]
        if joint:
            d["joint"] = joint
        if tip is not None:
            d["tip_proxy"] = tip
        self.doc["links"].append(d)
        return name

    def ignore(self, a, b):
        self.doc["ignore_collisions"].append([a, b])


def joint(name, parent, origin, axis, lo, hi):
    return {"name": name, "parent": parent, "origin": r6(origin), "axis": r6(axis), "lower": lo, "upper": hi}


def add_finger(spec, prefix, parent, mount, flex_axis, abd_axis, lengths, width, tip_r, abd_range, flex_ranges,
               extra_base=None):
    """Chain: [extra_base] -> knuckle (abduction, dummy) -> proximal -> middle -> distal(tip)."""
    links = []
    par, origin = parent, mount
    if extra_base is not None:
        eb_axis, eb_range, eb_len = extra_base
        name = spec.link(prefix + "_metacarpal", box(0, 0, 0.0, eb_len, width, width),
                         [([0, 0, 0.5 * eb_len], width * 1.1)],
                         joint(prefix + "_j5", par, origin, eb_axis, *eb_range))
        links.append(name)
        par, origin = name, [0, 0, eb_len]
    kn = spec.link(prefix + "_knuckle", box(0, 0, -0.002, 0.002, 0.002, 0.002), (),
                   joint(prefix + "_j4", par, origin, abd_axis, *abd_range))
    links.append(kn)
    par, origin = kn, [0, 0, 0]
    names = ("proximal", "middle", "distal")
    for i, (seg, (lo, hi)) in enumerate(zip(lengths, flex_ranges)):
        last = i == 2
        verts = box(0, 0, 0.0, seg * (0.75 if last else 1.0), width, width)
        if last:
            verts += tip_shell([0, 0, seg - tip_r], tip_r)
            prox = [([0, 0, 0.3 * seg], width * 1.05), ([0, 0, seg - tip_r], tip_r)]
            tip = 1
        else:
            prox = [([0, 0, 0.25 * seg], width * 1.1), ([0, 0, 0.75 * seg], width * 1.1)]
            tip = None
        name = spec.link(f"{prefix}_{names[i]}", verts, prox,
                         joint(f"{prefix}_j{3 - i}", par, origin, flex_axis, lo, hi), tip)
        links.append(name)
        par, origin = name, [0, 0, seg]
    # Self-collision among segments of one finger is exempt (adjacent-ish).
    for a in range(len(links)):
        for b in range(a + 1, len(links)):
            spec.ignore(links[a], links[b])
    spec.fingers[prefix] = links
    return links


def palm_link(spec, hx, hy, z0, z1, proxy_grid):
    prox = [([x, y, 0.5 * (z0 + z1)], r) for (x, y, r) in proxy_grid]
    return spec.link("palm", box(0, 0, z0, z1, hx, hy), prox)


def exempt_palm_near(spec, finger_links):
    for name in finger_links:
        if name.endswith(("knuckle", "proximal", "metacarpal")):
            spec.ignore("palm", name)


def four_finger_hand(name, seg, width, tip_r, spread, thumb_seg, palm, flex_hi=1.5, flip_thumb=True):
    """Allegro/Leap-like: index, middle, ring along +x, thumb opposite (-y)."""
    s = Spec(name)
    hx, hy = palm
    palm_link(s, hx, hy, -0.012, 0.008, [(x, y, 0.011) for x in (-0.02, 0.02) for y in (-0.02, 0.02)])
    fingers = []
    for i, fx in enumerate((-spread, 0.0, spread)):
        fingers.append(add_finger(s, f"f{i}", "palm", [fx, 0.7 * hy, 0.008], [1, 0, 0], [0, 1, 0], seg, width,
                                  tip_r, (-0.47, 0.47), [(-0.2, flex_hi), (-0.2, flex_hi), (-0.2, flex_hi)]))
    th = add_finger(s, "th", "palm", [0.0, -0.8 * hy, 0.008], [-1, 0, 0] if flip_thumb else [1, 0, 0], [0, 1, 0],
                    thumb_seg, width, tip_r, (0.26, 1.4), [(-0.2, 1.6), (-0.2, 1.7), (-0.2, 1.6)])
    fingers.append(th)
    for f in fingers:
        exempt_palm_near(s, f)
    return s.doc


def shadow_like():
    """22 DoF: thumb 5, index/middle/ring 4, little 5 (metacarpal), 5 tips."""
    s = Spec("shadow_like")
    hx, hy = 0.045, 0.05
    palm_link(s, hx, hy, -0.014, 0.008, [(x, y, 0.012) for x in (-0.03, 0.0, 0.03) for y in (-0.025, 0.025)])
    seg = (0.045, 0.025, 0.026)
    width, tip_r = 0.0095, 0.0105
    fingers = []
    for i, fx in enumerate((-0.033, -0.011, 0.011)):
        fingers.append(add_finger(s, f"f{i}", "palm", [fx, 0.7 * hy, 0.008], [1, 0, 0], [0, 1, 0], seg, width,
                                  tip_r, (-0.35, 0.35), [(-0.26, 1.57), (0.0, 1.57), (0.0, 1.57)]))
    fingers.append(add_finger(s, "lf", "palm", [0.033, 0.7 * hy, 0.0], [1, 0, 0], [0, 1, 0], seg, width, tip_r,
                              (-0.35, 0.35), [(-0.26, 1.57), (0.0, 1.57), (0.0, 1.57)],
                              extra_base=([0.3, 1, 0], (0.0, 0.79), 0.008)))
    fingers.append(add_finger(s, "th", "palm", [0.0, -0.8 * hy, 0.0], [-1, 0, 0], [0, 1, 0], (0.038, 0.032, 0.027),
                              width, tip_r, (-0.21, 1.2), [(0.0, 1.22), (-0.7, 0.7), (-0.26, 1.57)],
                              extra_base=([0, 0, 1], (-1.05, 1.05), 0.006)))
    for f in fingers:
        exempt_palm_near(s, f)
    return s.doc


def allegro_like():
    return four_finger_hand("allegro_like", (0.054, 0.038, 0.044), 0.0095, 0.012, 0.045, (0.05, 0.044, 0.044),
                            (0.055, 0.05))


def leap_like():
    return four_finger_hand("leap_like", (0.05, 0.036, 0.048), 0.011, 0.0125, 0.038, (0.046, 0.04, 0.05),
                            (0.05, 0.045), flex_hi=1.8)


# ----------------------------------------------------------------- objects
def obj_box(c, h):
    v = [(c[0] + sx * h[0], c[1] + sy * h[1], c[2] + sz * h[2]) for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]
    f = [(0, 2, 3), (0, 3, 1), (4, 5, 7), (4, 7, 6), (0, 1, 5), (0, 5, 4), (2, 6, 7), (2, 7, 3), (0, 4, 6), (0, 6, 2),
         (1, 3, 7), (1, 7, 5)]
    return v, f


def obj_capsule(c, axis, half_len, radius, n_seg=24, n_ring=8):
    """Closed convex capsule mesh along `axis` (0=x, 1=y, 2=z)."""
    rings = []
    for end, sign in ((-half_len, -1.0), (half_len, 1.0)):
        for k in range(n_ring + 1):
            phi = (math.pi / 2) * k / n_ring  # 0 at equator, pi/2 at pole
            if sign < 0:
                phi = -(math.pi / 2) + (math.pi / 2) * k / n_ring
            rings.append((end + radius * math.sin(phi), radius * math.cos(phi)))
    # rings ordered from -pole to +pole
    rings = sorted(set(rings))
    verts, faces = [], []
    ring_idx = []
    for (a, r) in rings:
        idx = []
        if r < 1e-9:
            verts.append((a, 0.0, 0.0))
            idx = [len(verts) - 1] * n_seg
        else:
            for s in range(n_seg):
                t = 2 * math.pi * s / n_seg
                verts.append((a, r * math.cos(t), r * math.sin(t)))
                idx.append(len(verts) - 1)
        ring_idx.append(idx)
    for i in range(len(ring_idx) - 1):
        A, B = ring_idx[i], ring_idx[i + 1]
        for s in range(n_seg):
            s1 = (s + 1) % n_seg
            if A[s] != A[s1]:
                faces.append((A[s], A[s1], B[s]))
            if B[s] != B[s1]:
                faces.append((A[s1], B[s1], B[s]))
    perm = {0: (0, 1, 2), 1: (1, 2, 0), 2: (1, 2, 0)}[axis]
    out = []
    for v in verts:
        p = [0.0, 0.0, 0.0]
        if axis == 0:
            p = [v[0], v[1], v[2]]
        elif axis == 1:
            p = [v[1], v[0], v[2]]
        else:
            p = [v[1], v[2], v[0]]
        out.append((c[0] + p[0], c[1] + p[1], c[2] + p[2]))
    del perm
    return out, faces


def drill_like_obj() -> str:
    """Config-2/4 object: 6 convex groups (capsule body, chuck, handle,
    battery, trigger, vent), about 1.4k hull faces at scale 0.10."""
    parts = [
        ("body", obj_capsule((0.0, 0.0, 0.35), 0, 0.55, 0.22, 24, 8)),
        ("chuck", obj_capsule((0.92, 0.0, 0.35), 0, 0.14, 0.11, 20, 6)),
        ("handle", obj_box((-0.1, 0.0, -0.2), (0.12, 0.1, 0.36))),
        ("battery", obj_box((-0.05, 0.0, -0.66), (0.3, 0.19, 0.1))),
        ("trigger", obj_box((0.1, 0.0, 0.02), (0.04, 0.05, 0.08))),
        ("grip", obj_capsule((-0.16, 0.0, -0.2), 2, 0.3, 0.1, 20, 6)),
    ]
    lines = ["# synthetic multi-part convex object (tools/gen_assets.py)"]
    offset = 0
    for name, (v, f) in parts:
        lines.append(f"g {name}")
        for p in v:
            lines.append("v %.9f %.9f %.9f" % p)
        for t in f:
            lines.append("f %d %d %d" % (t[0] + 1 + offset, t[1] + 1 + offset, t[2] + 1 + offset))
        offset += len(v)
    return "\n".join(lines) + "\n"


def main():
    (OUT / "hands").mkdir(parents=True, exist_ok=True)
    (OUT / "objects").mkdir(parents=True, exist_ok=True)
    for name, doc in (("allegro_like", allegro_like()), ("leap_like", leap_like()), ("shadow_like", shadow_like())):
        (OUT / "hands" / f"{name}.json").write_text(json.dumps(doc, indent=1) + "\n")
    (OUT / "objects" / "drill_like.obj").write_text(drill_like_obj())
    print("wrote", OUT)


if __name__ == "__main__":
    main()
