"""The oracle's suffix (layers s+1..e from layer s's output) composes with the prefix:
suffix(prefix_s(x), s, e) == prefix_e(x) exactly in fp64 (same per-layer definitions in the
same order), for block-structured archs and across the DenseNet transition / classifier
boundaries."""
import numpy as np
import pytest

import hapi_inputs
from oracle import prefix


@pytest.mark.parametrize("arch,s,e,size", [("resnet18", 4, 10, 64), ("densenet121", 5, 9, 64),
                                            ("alexnet", 13, 17, 224), ("vgg11", 5, 12, 64)])
def test_suffix_composes_with_prefix(arch, s, e, size):
    P = hapi_inputs.params(arch, 3)
    x = hapi_inputs.images(2, 4, size, size)
    a = prefix.prefix_forward(arch, P, x, s)
    want = prefix.prefix_forward(arch, P, x, e)
    got = prefix.suffix_forward(arch, P, a, s, e)
    assert got.shape == want.shape
    assert np.array_equal(got, want)
