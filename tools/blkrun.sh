# direct launches without programmatic dependent launch (graphs and PDL off) through the GPU suite
HAPI_GRAPH=0 HAPI_PDL=0 timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
