"""Per-level phase times of the level-loop merge (grid merge K2g at a G-rank,
MARSIT_FUSED_PROF build via MARSIT_SO): pass 1 + CTA scan, the exchange
(publish -> every CTA's total seen), pass 2 (draw offsets, coins, deposit),
CTA 0 of the launch, from %globaltimer."""
import ctypes as C
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06787_b200 import _native as N  # noqa: E402

L = N.lib()
L.marsit_debug_coop_prof.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 16)()
import runpy  # noqa: E402
L.marsit_debug_coop_prof(buf, 1)
sys.argv = ["bench_merge_rank.py"] + sys.argv[1:]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "bench_merge_rank.py"), run_name="__main__")
L.marsit_debug_coop_prof(buf, 0)
nl = max(buf[7], 1)
nk = max(buf[10], 1)
print(f"levels {buf[7]}: pass1+scan {buf[4]/nl/1e3:.2f} us, exchange {buf[5]/nl/1e3:.2f} us, pass2 {buf[6]/nl/1e3:.2f} us"
      f" | per launch ({buf[10]}): prologue {buf[8]/nk/1e3:.2f} us, CTA 0 start..end {buf[9]/nk/1e3:.2f} us")
