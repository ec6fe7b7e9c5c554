"""Coarse two-view geometry on the device against the reference's
estimate_fundamental_ransac (geometry.py:153-198): inlier masks identical,
F within 1e-6 (entries of the Frobenius-normalized matrix)."""

import os

import numpy as np
import pytest

from golden_io import GOLDEN

pytestmark = pytest.mark.gpu


def test_fransac_equals_reference():
    from paper_1512_06235_b200.fundamental import estimate_fundamental_ransac
    from paper_1512_06235_b200.types import InsufficientDataError

    z = np.load(os.path.join(GOLDEN, "fransac_cases.npz"))
    for k in range(int(z["n_cases"])):
        q, c, seed = z[f"c{k}_q"], z[f"c{k}_c"], int(z[f"c{k}_seed"])
        status = str(z[f"c{k}_status"])
        if status == "insufficient":
            with pytest.raises(InsufficientDataError):
                estimate_fundamental_ransac(q, c, seed=seed)
            continue
        if status == "overflow":
            with pytest.raises(OverflowError):
                estimate_fundamental_ransac(q, c, seed=seed)
            continue
        geom, mask = estimate_fundamental_ransac(q, c, seed=seed)
        np.testing.assert_array_equal(mask, z[f"c{k}_mask"], err_msg=f"case {k}")
        assert geom.inlier_count == int(z[f"c{k}_count"])
        assert geom.degenerate_planar == bool(z[f"c{k}_planar"]), k
        np.testing.assert_allclose(geom.F, z[f"c{k}_F"], atol=1e-6, err_msg=f"case {k}")
