"""The CUDA twin of the input generator is byte-identical to the numpy generator."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def test_images_match_numpy():
    import synth.gpu as sg
    for (H, W, unit0, n) in [(480, 640, 0, 1), (37, 53, 5, 3), (1080, 1920, 7, 1)]:
        g = sg.images(0, unit0, n, H, W).cpu().numpy()
        for k in range(n):
            assert (g[k] == synth.image(0, unit0 + k, H, W)).all(), (H, W, k)


def test_patches_match_numpy():
    import synth.gpu as sg
    g = sg.patches(2, 1000, 300).cpu().numpy()
    assert (g == synth.patches(2, range(1000, 1300))).all()
