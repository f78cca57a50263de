import os, sys
sys.path.insert(0, os.getcwd())
from tools.quick_time import run
for L in (2048, 4096, 8192):
    run(L, hc=8, kv=8, hs=64)
run(2048, hc=4, kv=4, hs=64)
