"""Print rel-L2 of the CUDA path vs the oracle for every split of several (arch, dtype,
size) cases.  Diagnostic companion of tests/test_gpu_parity.py (no asserts)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402
from tests.gpu_helpers import gpu_forward, oracle_all, rel_l2  # noqa: E402

CASES = [
    ("resnet18", "bf16", 64, 3), ("resnet18", "f32", 64, 3),
    ("alexnet", "f32", 224, 2), ("alexnet", "bf16", 224, 2),
    ("resnet50", "bf16", 96, 2), ("resnet50", "f32", 64, 2),
    ("vgg11", "bf16", 64, 2), ("vgg11", "f32", 64, 2),
    ("densenet121", "bf16", 64, 2), ("densenet121", "f32", 64, 2),
]
if len(sys.argv) > 1:
    CASES = [c for c in CASES if c[0] in sys.argv[1:] or c[1] in sys.argv[1:]]

print(H.build_info(), torch.cuda.get_device_name(0), flush=True)
for arch, act, sz, n in CASES:
    t0 = time.time()
    P = hapi_inputs.params(arch, 5)
    x = hapi_inputs.images(n, 6, sz, sz)
    L = H.hapi_num_layers(arch)
    try:
        model = H.Model(arch, act, list(P.values()), n, 1, L, in_h=sz, in_w=sz)
    except Exception as e:  # noqa: BLE001
        print(f"{arch} {act} {sz}: create failed: {e}", flush=True)
        continue
    ref = oracle_all(arch, 5, 6, n, sz, sz)
    errs = []
    for s in range(1, L + 1):
        try:
            got, _ = gpu_forward(arch, act, s, x, P, model=model)
            errs.append(f"{s}:{rel_l2(got, ref[s - 1].reshape(n, -1)):.1e}")
        except Exception as e:  # noqa: BLE001
            errs.append(f"{s}:ERR({str(e)[:80]})")
            break
    print(f"{arch:12s} {act:5s} {sz:4d} n={n} [{time.time() - t0:.0f}s] " + " ".join(errs), flush=True)
    model.close()
