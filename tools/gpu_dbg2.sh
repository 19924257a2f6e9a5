MT_NVCC_EXTRA="-DMT_BREADCRUMBS -DMT_SPIN_TIMEOUT_CYCLES=(1ull<<30)" python -c "from paper_2510_18830_b200 import build; build.build()"
MT_NVCC_EXTRA="-DMT_BREADCRUMBS -DMT_SPIN_TIMEOUT_CYCLES=(1ull<<30)" timeout 120 python tools/debug_csr.py 2>&1 | tail -30
