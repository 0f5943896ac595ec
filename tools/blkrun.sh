# stem epilogue without spills (bias as kernel parameter) vs the previous build: parity, bitwise, layer time
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "every_split_224 or configs_2_3" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_fusion_bits.py -q -k "STEM" 2>&1 | tail -1
python - <<'PY'
import os, subprocess, sys, numpy as np
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import hapi_inputs
from tests.gpu_helpers import gpu_forward
for arch, s, sz in (("resnet50", 2, 224), ("densenet121", 2, 224), ("resnet18", 4, 160)):
    P = hapi_inputs.params(arch, 5); x = hapi_inputs.images(3, 6, sz, sz)
    y, m = gpu_forward(arch, "bf16", s, x, P); m.close()
    np.save(f"/tmp/stem_{arch}.npy", y)
'''
outs = {}
for lib in ("paper_2210_08650_b200/libhapi.so", "abtest/libhapi_stemold.so"):
    env = dict(os.environ, HAPI_LIB=lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    outs[lib] = {a: np.load(f"/tmp/stem_{a}.npy") for a in ("resnet50", "densenet121", "resnet18")}
a, b = outs.values()
print("stem bitwise equal:", all(np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)) for k in a))
PY
for r in 1 2; do
for lib in paper_2210_08650_b200/libhapi.so abtest/libhapi_stemold.so; do
  HAPI_LIB=$lib timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/stem_ab.txt 2>&1
  echo "$lib: $(head -1 gpurun_out/stem_ab.txt | cut -c1-80) | $(grep -h 'conv1.weight 4x4' gpurun_out/stem_ab.txt | cut -c1-30)"
done
done
