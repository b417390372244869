"""Diagnose mesh-stage gradient differences in the trajectory parity run: for every
(snapshot, grasp) whose GPU gradient differs from the oracle's, check whether the device FK
is bitwise the oracle's, and compare the GPU pair kernel with the oracle's signed_distance on
identical poses (the device's own FK). Writes gpurun_out/diag_trajectory.json."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2412_16490_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_gpu_parity import gpu_pairs, gpu_fcq  # noqa: E402
from test_gpu_trajectory import SNAPS  # noqa: E402


def world_colmajor_to_pose(w):
    return w  # (L, 12) R column-major + t: the pair surfaces' pose layout


def main():
    out = {}
    eng = G.Engine(0)
    cases = [("config2", G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/shadow_like.json"),
              G.load_object(ROOT / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)),
             ("config1_sphere", G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/allegro_like.json"),
              G.make_primitive("sphere", 0.08))]
    for name, hand, obj in cases:
        eng.set_hand(hand)
        eng.set_object(obj)
        cfg = G.RunConfig()
        cfg.batch, cfg.seed = 64, 17
        x0 = G.init_poses(hand, obj, 64, 17, cfg.init)
        _, T = eng.synthesize_traced(cfg, x0, SNAPS)
        rows = []
        L, P = hand.n_links, obj.n_parts
        for k, (s, it) in enumerate(SNAPS):
            if s == 0:
                continue
            x_in = T["x_in"][k]
            e_ref, g_ref = O.total_energy(hand, obj, cfg, s, x_in, anchors=T["anchors"][k])
            gerr = np.abs(T["grad"][k] - g_ref).max(axis=1) / np.maximum(np.abs(g_ref).max(axis=1), 1e-300)
            for g in np.where(gerr > 1e-9)[0]:
                w_gpu = T["world_in"][k][g]
                w_ref = O.forward_kinematics(hand, x_in[g:g + 1])[0]
                fk_bitwise = bool((w_gpu == w_ref).all())
                links = np.repeat(np.arange(L), P)
                parts = np.tile(np.arange(P), L)
                poses = np.repeat(w_gpu, P, axis=0)
                ref_same = O.signed_distance(hand, obj, links, parts, poses)
                got_same = gpu_pairs(eng, links, parts, poses)
                diff_same = np.abs(ref_same[:, :10] - got_same[:, :10]).max(axis=1) > 0
                ref_own = O.signed_distance(hand, obj, links, parts, np.repeat(w_ref, P, axis=0))
                diff_fk = np.abs(ref_own[:, :10] - ref_same[:, :10]).max(axis=1) > 0
                fq_g = gpu_fcq(eng, hand, x_in[g:g + 1])[0]
                fq_o = O.fine_contact_query(hand, obj, x_in[g:g + 1])[0]
                rows.append(dict(stage=s, iter=it, grasp=int(g), grad_err=float(gerr[g]),
                                 energy_err=float(abs(T["energy"][k][g] - e_ref[g]) / abs(e_ref[g])),
                                 fk_bitwise=fk_bitwise, fk_maxdiff=float(np.abs(w_gpu - w_ref).max()),
                                 pairs_differ_same_poses=int(diff_same.sum()),
                                 pairs_differ_same_poses_epa=[int(v) for v in ref_same[diff_same, 10]],
                                 pairs_differ_same_poses_max=float(np.abs(ref_same[:, :10] - got_same[:, :10]).max()),
                                 pairs_changed_by_fk_ulps=int(diff_fk.sum()),
                                 fcq_maxdiff=float(np.abs(fq_g - fq_o).max())))
        out[name] = rows
        print(name, json.dumps(rows, indent=None)[:3000])
    dst = ROOT / "gpurun_out"
    dst.mkdir(exist_ok=True)
    (dst / "diag_trajectory.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
