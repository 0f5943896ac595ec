"""The seeded generator's parameter table equals torchvision's state_dict (library pin)."""
import numpy as np
import pytest
import torchvision

import hapi_inputs

TV = {"alexnet": torchvision.models.alexnet, "resnet18": torchvision.models.resnet18,
      "resnet50": torchvision.models.resnet50, "vgg11": torchvision.models.vgg11,
      "densenet121": torchvision.models.densenet121}


@pytest.mark.parametrize("arch", hapi_inputs.ARCHS)
def test_param_table_matches_torchvision(arch):
    sd = TV[arch](weights=None).state_dict()
    want = [(k, tuple(v.shape)) for k, v in sd.items() if not k.endswith("num_batches_tracked")]
    got = [(n, s) for n, s, _ in hapi_inputs.param_table(arch)]
    assert got == want


def test_generators_deterministic():
    a = hapi_inputs.images(2, 1)
    b = hapi_inputs.images(2, 1)
    assert a.dtype == np.float32 and a.shape == (2, 3, 224, 224)
    np.testing.assert_array_equal(a, b)
    p1 = hapi_inputs.params("resnet18", 7)
    p2 = hapi_inputs.params("resnet18", 7)
    for k in p1:
        np.testing.assert_array_equal(p1[k], p2[k])
        assert p1[k].dtype == np.float32 and p1[k].flags.c_contiguous
    assert p1["bn1.running_var"].min() >= 0.8
