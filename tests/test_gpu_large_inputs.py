"""Larger inputs (iNaturalist-like ~2x and PlantLeaves-like ~8x images,
PAPER.md:94-157): the same plans at 448x448 / 640x640 / odd sizes, checked against the
oracle on a couple of images.  Exercises the size-dependent kernel choices: more stem strips
in the stem+pool kernel, halo tiles of one row (112-wide maps), im2col for maps wider than a
halo tile (160-wide), non-multiple-of-tile M."""
import numpy as np
import pytest

import hapi_inputs
from tests.gpu_helpers import gpu_forward, oracle_all
from tests.parity_check import check_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("arch,act,split,size,n", [
    ("resnet50", "bf16", 21, 448, 2),
    ("resnet50", "bf16", 9, 640, 1),
    ("densenet121", "bf16", 9, 320, 2),
    ("resnet18", "bf16", 10, 288, 3),
    ("vgg11", "bf16", 11, 288, 2),
    ("resnet18", "f32", 8, 384, 2),
])
def test_large_inputs_match_oracle(arch, act, split, size, n):
    P = hapi_inputs.params(arch, 41)
    x = hapi_inputs.images(n, 42, size, size)
    got, m = gpu_forward(arch, act, split, x, P)
    m.close()
    ref = oracle_all(arch, 41, 42, n, size, size, upto=split)[split - 1]
    check_close(got, ref, act, f"{arch} s={split} {size}px")
