"""MHA (kv == hc) forward timing at small and large L (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_time import run  # noqa: E402

for L in (4096, 8192, 16384):
    run(L, hc=8, kv=8, hs=64)
run(32768, hc=8, kv=8, hs=128)
run(32768, hc=12, kv=4, hs=128)   # odd GQA group (3)
