# the layer-at-a-time plan (fused blocks off) through the whole GPU suite
HAPI_BLOCK=0 timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
