"""Native model snapshot reader (msfm.io.read_model io.py:51-84) against the
reference's own read_model on its write_model output (tests/golden/model_io,
make_golden_model_io.py): contents, and FormatError text for malformed files."""

import json
import os

import numpy as np
import pytest

from golden_io import GOLDEN

D = os.path.join(GOLDEN, "model_io")


@pytest.mark.parametrize("name", ["holdout", "c1"])
def test_snapshot_arrays_and_model_equal_reference(name):
    from paper_1512_06235_b200.model_io import read_model, read_snapshot

    z = np.load(os.path.join(D, f"{name}.npz"))
    arr = read_snapshot(os.path.join(D, f"{name}.msfm"))
    order = np.argsort(arr.cam_id)
    np.testing.assert_array_equal(arr.cam_id[order], z["cam_id"])
    np.testing.assert_array_equal(arr.K[order], z["K"])
    np.testing.assert_array_equal(arr.R[order], z["R"])
    np.testing.assert_array_equal(arr.t[order], z["t"])
    np.testing.assert_array_equal(arr.point_xyz, z["xyz"])
    pid = np.repeat(np.arange(len(arr.point_xyz)), np.diff(arr.track_ptr))
    np.testing.assert_array_equal(np.stack([pid, arr.track_img, arr.track_fid], 1), z["track"])
    assert arr.stage_tag == str(z["stage"])
    m = read_model(os.path.join(D, f"{name}.msfm"))
    assert m.stage_tag == str(z["stage"])
    assert m.image_ids() == z["cam_id"].tolist()
    assert sorted(m.points) == list(range(len(z["xyz"])))
    np.testing.assert_array_equal(np.stack([m.points[p].position for p in sorted(m.points)]), z["xyz"])


def test_malformed_files_raise_the_reference_messages():
    from paper_1512_06235_b200 import types
    from paper_1512_06235_b200.model_io import read_model

    exp = json.load(open(os.path.join(D, "expected.json")))
    for name, msg in exp.items():
        path = os.path.join(D, f"bad_{name}.msfm")
        if msg is None:
            read_model(path)
            continue
        with pytest.raises(types.FormatError) as ei:
            read_model(path)
        assert str(ei.value) == msg.replace("<path>", path), name
