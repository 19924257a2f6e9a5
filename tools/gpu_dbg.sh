python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 300 python tools/debug_fwd_ring.py 2 2>&1 | tail -20
