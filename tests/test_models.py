"""CPU tests: load-time models (hull, objects, hand spec) against the
reference's own test expectations (proj/tests/test_geometry.cpp,
test_object.cpp, test_hand.cpp)."""
import json

import numpy as np
import pytest


def three_box_obj() -> str:
    """test_pipeline.cpp:64-87: three separated boxes as one OBJ."""
    lines, offset = [], 0
    faces = [(0, 2, 3), (0, 3, 1), (4, 5, 7), (4, 7, 6), (0, 1, 5), (0, 5, 4), (2, 6, 7), (2, 7, 3), (0, 4, 6),
             (0, 6, 2), (1, 3, 7), (1, 7, 5)]
    for name, c, h in (("a", (-0.8, 0.0, 0.0), (0.4, 0.5, 0.6)), ("b", (0.9, 0.1, -0.2), (0.5, 0.4, 0.3)),
                       ("c", (0.1, 0.9, 0.5), (0.3, 0.3, 0.4))):
        lines.append(f"g {name}")
        for sx in (-1, 1):
            for sy in (-1, 1):
                for sz in (-1, 1):
                    lines.append(f"v {c[0] + sx * h[0]} {c[1] + sy * h[1]} {c[2] + sz * h[2]}")
        for t in faces:
            lines.append(f"f {offset + t[0] + 1} {offset + t[1] + 1} {offset + t[2] + 1}")
        offset += 8
    return "\n".join(lines) + "\n"


def box_points(hx, hy, hz):
    return [(sx * hx, sy * hy, sz * hz) for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]


def euler_characteristic(verts, faces):
    edges = set()
    for t in faces:
        for e in range(3):
            u, v = int(t[e]), int(t[(e + 1) % 3])
            edges.add((min(u, v), max(u, v)))
    return len(verts) - len(edges) + len(faces)


def test_builtin_trident_structure(trident):
    # test_hand.cpp:254-289: 7 links, 6 joints, 3 tips, 15 link pairs.
    assert trident.n_links == 7 and trident.dof() == 6 and trident.n_tips == 3
    assert trident.n_pairs == 15
    assert len(trident.proxies) == 19
    assert list(np.diff(trident.link_vert_begin)) == [12, 8, 57, 8, 57, 8, 57]
    assert list(np.diff(trident.link_face_begin)) == [20, 12, 110, 12, 110, 12, 110]
    np.testing.assert_array_equal(trident.lower, [-0.35, -0.2] * 3)
    np.testing.assert_array_equal(trident.upper, [1.40, 1.50] * 3)


def test_builtin_json_round_trips(G, trident):
    text = G.builtin_hand_json()
    doc = json.loads(text)
    assert doc["format_version"] == 1 and doc["name"] == "trident"
    again = G.HandModel.from_json(text)
    assert again.n_pairs == trident.n_pairs
    np.testing.assert_array_equal(again.proxies, trident.proxies)


def test_hand_spec_errors(G):
    bad = [
        "{not json",
        json.dumps({"format_version": 2, "links": []}),
        json.dumps({"format_version": 1, "links": []}),
        json.dumps({"format_version": 1, "links": [{"name": "a", "vertices": [[0, 0, 0], [1, 0, 0], [0, 1, 0]]}]}),
    ]
    for text in bad:
        with pytest.raises(G.HandError):
            G.HandModel.from_json(text)


@pytest.mark.parametrize("name,nv,nf", [("sphere", 162, 320), ("box", 8, 12), ("cylinder", 64, 124),
                                        ("capsule", 118, 232), ("flat_box", 8, 12)])
def test_primitives_normalize(G, name, nv, nf):
    # object.cpp:212-235 + test_object.cpp:229-274: bbox diagonal 2*scale,
    # gravity center at the origin, hull counts from SURVEY 8.
    for scale in (0.06, 0.1):
        o = G.make_primitive(name, scale)
        assert o.n_parts == 1
        assert len(o.verts) == nv and len(o.faces) == nf
        assert o.bbox_diagonal == pytest.approx(2 * scale, rel=1e-12)
        assert np.linalg.norm(o.mass_center) < 1e-12
        assert euler_characteristic(o.verts, o.faces) == 2
        assert o.source == "builtin:" + name


def test_noisy_cube_hull_keeps_corners(G):
    # test_geometry.cpp:38-61.
    rng = np.random.default_rng(7)
    cloud = np.array(box_points(0.5, 0.5, 0.5) + list(rng.uniform(-0.49, 0.49, size=(200, 3))))
    o = G.ObjectModel.from_points([cloud])
    assert len(o.verts) == 8
    assert o.part_volume[0] == pytest.approx(1.0, rel=1e-12)
    assert np.linalg.norm(o.part_centroid[0]) < 1e-12


def test_degenerate_hulls_rejected(G):
    planar = [(i * 0.1, j * 0.1, 0.0) for i in range(5) for j in range(5)]
    for pts in (planar, [(0, 0, 0), (1, 0, 0), (0, 1, 0)], [(0.3, -0.2, 0.9)] * 50):
        with pytest.raises(G.GeometryError):
            G.ObjectModel.from_points([np.array(pts, dtype=float)])


def test_near_duplicates_merge(G):
    pts = []
    for c in box_points(0.5, 0.5, 0.5):
        pts.append(c)
        pts.append(tuple(np.array(c) + 1e-13))
    assert len(G.ObjectModel.from_points([np.array(pts)]).verts) == 8


def test_tetra_volume_centroid(G):
    o = G.ObjectModel.from_points([np.array([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], dtype=float)])
    assert o.part_volume[0] == pytest.approx(1 / 6, rel=1e-14)
    np.testing.assert_allclose(o.part_centroid[0], [0.25] * 3, atol=1e-13)


def test_obb_is_tight_on_boxes(G):
    # test_geometry.cpp:135-145.
    o = G.ObjectModel.from_points([np.array(box_points(0.5, 0.2, 0.1))])
    obb = o.part_obb[0]
    assert np.linalg.norm(obb[:3]) < 1e-12
    np.testing.assert_allclose(sorted(obb[3:6], reverse=True), [0.5, 0.2, 0.1], atol=1e-10)


def test_three_box_object_parses(G):
    o = G.parse_object_text(three_box_obj(), 0.12, "three_boxes")
    assert o.n_parts == 3
    assert o.bbox_diagonal == pytest.approx(0.24, rel=1e-12)


def test_nonconvex_group_rejected(G):
    # test_object.cpp:140-163: an L-shaped group fails the 5% screen by name.
    pts = [(0, 0, 0), (2, 0, 0), (2, 1, 0), (1, 1, 0), (1, 2, 0), (0, 2, 0)]
    lines = ["g ell"] + [f"v {x} {y} {z}" for (x, y, z) in pts] + [f"v {x} {y} 1" for (x, y, _) in pts]
    bottom = [(1, 3, 2), (1, 4, 3), (1, 5, 4), (1, 6, 5)]
    top = [(7, 8, 9), (7, 9, 10), (7, 10, 11), (7, 11, 12)]
    sides = []
    for i in range(6):
        a, b = i + 1, (i + 1) % 6 + 1
        sides += [(a, b, b + 6), (a, b + 6, a + 6)]
    for t in bottom + top + sides:
        lines.append("f %d %d %d" % t)
    with pytest.raises(G.ObjectError, match="ell"):
        G.parse_object_text("\n".join(lines), 0.1, "ell")


def test_object_parse_errors(G):
    for text in ("", "v 0 0 0\nf 1 2 3\n", "v a b c\n"):
        with pytest.raises(G.ObjectError):
            G.parse_object_text(text, 0.1, "bad")
