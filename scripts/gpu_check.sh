python scripts/level_times.py 2>&1 | tail -9
CUTFEM_CLUSTER_MAX=100000 python scripts/level_times.py 2>&1 | tail -9
