"""Print a workload's launch plan (hapi_plan_describe).  Usage: python tools/plan_dump.py arch split size [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402

arch, split, size = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
batch = int(sys.argv[4]) if len(sys.argv) > 4 else 2
P = list(hapi_inputs.params(arch, 1).values())
m = H.Model(arch, "bf16", P, batch, split, split, in_h=size, in_w=size)
info = m.plan_info(split)
for i, d in enumerate(info["desc"]):
    print(f"{i:3d} {info['bytes'][i] / 1e6:9.3f} MB/img  {d}")
m.close()
