"""Per-rank attention shapes of the N=8 configurations, timed alone on one
GPU (development aid): what one rank's kernel does at c2/c3/c4/c5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_time import run  # noqa: E402

run(32768, hc=4, kv=1)                   # c2 U8R1: full L, 4 local q heads, 1 kv head
run(16384, hc=32, kv=8, causal=False)    # c3 U1R8: one off-diagonal ring step ~ 16K x 16K dense
run(32768, hc=8, kv=2, causal=False)     # c4-like step at reduced L (U4: 8 local heads)
run(32768, hc=8, kv=1)                   # c5 U4R2 kv4: 8 local q heads, 1 kv head
