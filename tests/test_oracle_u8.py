"""Pins of the oracle's u8 ingest (oracle.prefix.normalize_u8): torchvision's own Normalize on
ToTensor-scaled images, per-channel placement, and the identity case."""
import numpy as np
import pytest
import torch

import hapi_inputs
from oracle import prefix


def test_matches_torchvision_normalize():
    from torchvision.transforms import functional as F
    u8 = hapi_inputs.images_u8(2, 5, 16, 12)
    mean, std = [0.485, 0.456, 0.406], [0.229, 0.224, 0.225]
    scale = [1.0 / (255.0 * s) for s in std]
    shift = [-m / s for m, s in zip(mean, std)]
    got = prefix.normalize_u8(u8, scale, shift)
    want = torch.stack([F.normalize(torch.from_numpy(im).double() / 255.0, mean, std) for im in u8]).numpy()
    assert np.allclose(got, want, rtol=0, atol=1e-12)


def test_per_channel_placement_and_identity():
    u8 = np.ones((1, 3, 2, 2), np.uint8)
    x = prefix.normalize_u8(u8, [1.0, 2.0, 3.0], [10.0, 20.0, 30.0])
    assert x[0, :, 0, 0].tolist() == [11.0, 22.0, 33.0]          # channel c uses scale[c], shift[c]
    u8 = hapi_inputs.images_u8(1, 6, 4, 4)
    assert np.array_equal(prefix.normalize_u8(u8, [1.0] * 3, [0.0] * 3), u8.astype(np.float64))
    assert u8.min() >= 0 and u8.max() <= 255 and u8.dtype == np.uint8


def test_rejects_non_u8():
    with pytest.raises(ValueError):
        prefix.normalize_u8(np.zeros((1, 3, 2, 2), np.float32), [1.0] * 3, [0.0] * 3)
