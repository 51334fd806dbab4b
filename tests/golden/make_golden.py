"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref: the reference's own
hot-path headers under /root/reference, compiled against oracle/eigen_shim by oracle/Makefile).

Run in the build container (needs /root/reference for the first build of oracle/_ref):
    python tests/golden/make_golden.py
Each fixture holds the inputs (seeded numpy draws) and the reference's fp32 outputs: per-splat
fields, sorted refs, tile offsets, image, stats, and the reference's (DC-only) gradients for a
fixed dL/dimage.
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_2409_04751_b200 import Camera, Scene, synthetic  # noqa: E402


def spherical_scene(n, seed, sh_rest=0.2):
    r = np.random.default_rng(seed)
    th, ph = r.uniform(0.05, 2.8, n), r.uniform(0, 2 * math.pi, n)
    d = r.uniform(1.5, 6.0, n)
    means = d[:, None] * np.stack([np.sin(th) * np.cos(ph), np.cos(th), np.sin(th) * np.sin(ph)], 1)
    means[:, [1, 2]] = means[:, [2, 1]]
    ls = np.log(r.uniform(0.03, 0.25, (n, 3)))
    q = r.standard_normal((n, 4))
    p = r.uniform(0.05, 0.95, n)
    sh = np.zeros((n, 48))
    sh[:, [0, 16, 32]] = r.uniform(-1.2, 1.2, (n, 3))
    sh += r.uniform(-sh_rest, sh_rest, (n, 48)) * (np.arange(48) % 16 != 0)
    f = lambda a: np.ascontiguousarray(a, np.float32)
    return Scene(f(means), f(q), f(ls), f(np.log(p / (1 - p))), f(sh), np.array([0.1, 0.15, 0.2], np.float32))


def cases():
    s = spherical_scene(800, 1)
    yield "fisheye_sh3", s, Camera.fisheye(160, 120, 40.0, 40.0, 80.0, 60.0).as_float32(), 3
    s, _, _, _ = synthetic.config(3, n=2500)
    s.means = (s.means / 3.0).astype(np.float32)
    s.log_scales = (s.log_scales + 1.0).astype(np.float32)
    rng = np.random.default_rng(5)
    r_wc, t_wc = synthetic.random_pose(rng, box=1.0)
    cam = Camera.fisheye(192, 128, 0.5 * math.hypot(192, 128) / math.radians(95), 0.5 * math.hypot(192, 128) /
                         math.radians(95), 96.0, 64.0, math.radians(95))
    cam.rotation_wc, cam.translation_wc = r_wc, t_wc
    yield "fisheye_rotated_95deg", s, cam.as_float32(), 3
    s, deg, cams, _ = synthetic.config(0, n=2000)
    yield "cfg0_subset", s, cams[0], deg


def golden_dl(cam):
    """dL/dimage used for every fixture (regenerated from its seed, not stored)."""
    return np.random.default_rng(123).standard_normal((cam.height, cam.width, 3)).astype(np.float32)


def main():
    oracle.build()
    assert oracle.ref_available(), "oracle/_ref not built (needs /root/reference)"
    for name, scene, cam, deg in cases():
        res = oracle.render(scene, cam, sh_degree=deg, impl="ref", threads=4)
        dl = golden_dl(cam)
        grads, sg = oracle.backward(res, scene.n, dl, want_splat_grads=True)
        st = res.stats()
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"),
            means=scene.means, rotations=scene.rotations, log_scales=scene.log_scales,
            opacity_logits=scene.opacity_logits, sh=scene.sh, background=scene.background,
            camera=cam.to_array(), sh_degree=deg,
            mean_px=res.get("mean_px"), conic=res.get("conic"), depth=res.get("depth"), radius=res.get("radius"),
            color=res.get("color"), alpha=res.get("alpha"), source=res.get("source"), refs=res.get("refs"),
            offsets=res.get("offsets"), image=res.image, grads=grads, splat_grads=sg,
            stats=np.array([st["num_intersections"], st["num_splats"], st["num_culled"], st["num_degenerate"]]))
        print(name, "I=%d splats=%d" % (res.num_intersections, res.num_splats))


if __name__ == "__main__":
    main()
