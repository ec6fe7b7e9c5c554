"""Golden model snapshots and error cases from the REFERENCE (msfm.io, io.py:16-84).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_model_io.py

Writes tests/golden/model_io/{holdout,c1}.msfm with the reference's write_model,
their read_model() contents as npz, and malformed variants with the exact
FormatError text read_model raises (expected.json; paths are relative).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "model_io")
sys.path.insert(0, os.environ.get("MSFM_REF_PATH", "/root/reference/pkg/src"))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from msfm.errors import FormatError  # noqa: E402
from msfm.io import read_model, write_model  # noqa: E402
from msfm.synth import SceneSpec, generate_scene  # noqa: E402

from make_golden_localize import partial_model  # noqa: E402


def dump(name, model):
    path = os.path.join(OUT, f"{name}.msfm")
    write_model(model, path)
    m = read_model(path)
    ids = m.image_ids()
    pids = m.point_ids()
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"),
                        stage=np.array(m.stage_tag), cam_id=np.array(ids),
                        K=np.stack([m.cameras[i].K for i in ids]), R=np.stack([m.cameras[i].R for i in ids]),
                        t=np.stack([m.cameras[i].t for i in ids]),
                        xyz=np.stack([m.points[p].position for p in pids]),
                        track=np.array([[p, i, f] for p in pids for i, f in m.points[p].track.items()]))
    return path


def bad_cases(src):
    lines = open(src).read().splitlines()
    cam = next(k for k, l in enumerate(lines) if l.startswith("CAM"))
    pt = next(k for k, l in enumerate(lines) if l.startswith("PT"))
    lines = lines[:pt + 3]                   # header, stage, cameras, three points
    c = lines[cam].split()
    p = lines[pt].split()
    cases = {
        "no_header": ["MSFM-MODEL 2"] + lines[1:],
        "empty": [],
        "unknown_record": lines[:pt] + ["XYZ 1 2 3"] + lines[pt:],
        "bad_float_cam": lines[:cam] + [" ".join(c[:3] + ["1.0.0"] + c[4:])] + lines[cam + 1:],
        "bad_int_cam": lines[:cam] + [" ".join(["CAM", "x7"] + c[2:])] + lines[cam + 1:],
        "short_cam": lines[:cam] + [" ".join(c[:4])] + lines[cam + 1:],
        "short_R": lines[:cam] + [" ".join(c[:10])] + lines[cam + 1:],
        "short_t": lines[:cam] + [" ".join(c[:15])] + lines[cam + 1:],
        "bad_det": lines[:cam] + [" ".join(c[:5] + [repr(2.0 * float(v)) for v in c[5:8]] + c[8:])]
                   + lines[cam + 1:],
        "dup_cam": lines[:cam + 1] + [lines[cam]] + lines[cam + 1:],
        "pt_missing_len": lines[:pt] + [" ".join(p[:4])] + lines[pt + 1:],
        "pt_short_track": lines[:pt] + [" ".join(p[:5] + p[5:7])] + lines[pt + 1:],
        "pt_one_view": lines[:pt] + [" ".join(p[:4] + ["1"] + p[5:7])] + lines[pt + 1:],
        "pt_unregistered": lines[:pt] + [" ".join(p[:5] + ["999"] + p[6:])] + lines[pt + 1:],
        "pt_owned": lines[:pt + 1] + [lines[pt]] + lines[pt + 1:],
        "pt_bad_fid": lines[:pt] + [" ".join(p[:6] + ["1e3"] + p[7:])] + lines[pt + 1:],
        "crlf_and_blank": ["MSFM-MODEL 1", "", "   "] + lines[1:],
    }
    out = {}
    for name, ls in cases.items():
        path = os.path.join(OUT, f"bad_{name}.msfm")
        with open(path, "w", newline="") as f:
            f.write(("\r\n" if name == "crlf_and_blank" else "\n").join(ls) + ("\n" if ls else ""))
        try:
            read_model(path)
            out[name] = None
        except FormatError as exc:
            out[name] = str(exc).replace(path, "<path>")
    return out


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    hold = generate_scene(SceneSpec(n_cameras=12, n_points=700, visibility_fraction=0.7,
                                    pixel_noise=0.3, descriptor_noise=3.0, seed=77))
    m = partial_model(hold, range(9))
    m.stage_tag = "coarse"
    src = dump("holdout", m)
    c1 = generate_scene(SceneSpec(n_cameras=20, n_points=2000, visibility_fraction=0.6,
                                  pixel_noise=0.5, descriptor_noise=4.0, seed=1))
    dump("c1", c1.ground_truth_model())
    exp = bad_cases(src)
    with open(os.path.join(OUT, "expected.json"), "w") as f:
        json.dump(exp, f, indent=1, sort_keys=True)
    print(json.dumps(exp, indent=1))
