"""Load-time convex parts on the device (grasp_build_convex_parts): the device
quickhull + make_convex_part (geometry.cpp:414-466, hull3d.cpp:291-303) must reproduce the host
builder (ObjectModel.from_points) bit for bit: vertex order, face order, volume, centroid and the
PCA box, on the drill mesh's groups, the primitives, random clouds, lattices full of coplanar
and collinear points, and near-duplicate points inside the merge tolerance."""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def obj_groups(path):
    verts, groups, cur = [], {}, None
    for line in Path(path).read_text().splitlines():
        t = line.split()
        if not t or t[0].startswith("#"):
            continue
        if t[0] == "v":
            verts.append([float(x) for x in t[1:4]])
        elif t[0] in ("g", "o"):
            cur = t[1]
            groups.setdefault(cur, set())
        elif t[0] == "f":
            cur = cur or "default"
            groups.setdefault(cur, set()).update(int(x.split("/")[0]) - 1 for x in t[1:])
    verts = np.array(verts)
    return [verts[sorted(ix)] for ix in groups.values()]


def clouds():
    rng = np.random.default_rng(3)
    out = obj_groups(ROOT / "paper_2412_16490_b200/assets/objects/drill_like.obj")
    import paper_2412_16490_b200 as G
    for name in ("sphere", "box", "cylinder", "capsule", "flat_box"):
        o = G.make_primitive(name, 0.1)
        out.append(o.part_vertices(0))
    for n in (8, 50, 200, 1000):
        out.append(rng.normal(size=(n, 3)) * 0.05)
    d = rng.normal(size=(600, 3))
    out.append(0.03 * d / np.linalg.norm(d, axis=1)[:, None])
    g = np.stack(np.meshgrid(*[np.linspace(-0.02, 0.02, 5)] * 3, indexing="ij"), -1).reshape(-1, 3)
    out.append(g)                                    # lattice: coplanar/collinear everywhere
    out.append(np.concatenate([g, g + 3e-10, g[::7]]))  # duplicates within the merge tolerance
    out.append(rng.integers(-3, 4, size=(300, 3)) * 0.01)  # integer lattice with repeats
    return out


def test_device_convex_parts_bitwise_equal_host_builder():
    import paper_2412_16490_b200 as G
    parts = clouds()
    dev = G.build_convex_parts(parts)
    assert len(dev) == len(parts)
    for i, (pts, d) in enumerate(zip(parts, dev)):
        assert d["status"] == 0, i
        host = G.ObjectModel.from_points([pts])
        assert np.array_equal(d["vertices"], host.part_vertices(0)), i
        assert np.array_equal(d["faces"], host.part_faces(0)), i
        assert d["volume"] == host.part_volume[0], i
        assert np.array_equal(d["centroid"], host.part_centroid[0]), i
        assert np.array_equal(d["obb"], host.part_obb[0]), i


def test_device_convex_parts_degenerate_inputs():
    import paper_2412_16490_b200 as G
    flat = np.c_[np.random.default_rng(1).normal(size=(40, 2)), np.zeros(40)]
    line = np.outer(np.linspace(0, 1, 10), [1.0, 2.0, 3.0])
    few = np.eye(3)
    res = G.build_convex_parts([flat, line, few, np.random.default_rng(2).normal(size=(30, 3))])
    assert [r["status"] for r in res] == [1, 1, 1, 0]
    for pts in (flat, line, few):
        with pytest.raises(G.GeometryError):
            G.ObjectModel.from_points([pts])
    assert G.build_convex_parts([]) == []
