"""hs=64 forward timing (development aid): python tools/time_hs64.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_time import run  # noqa: E402

for L in (8192, 32768):
    run(L, hc=8, kv=8, hs=64)
run(32768, hc=32, kv=8, hs=64)
