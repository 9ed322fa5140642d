"""Do DFMA and DMMA share the FP64 issue capacity?  Times k_mix (k_probe.cu):
all warps DFMA (T0), all warps m8n8k4 DMMA (T1), half/half (T2), with the
per-warp work balanced so T0 ~ T1.  T2 ~ T0: one shared pipe; T2 ~ T0/2: two."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_08284_b200 as ankh  # noqa: E402

lib = ankh.lib()
it_f, it_m = 2048, 4096  # 4096 FMA per warp-iteration each (DFMA 128 x 32, DMMA 8 x 256 ... x2)
for rep in range(2):
    t = [lib.ankh_probe_fp64_mix_ms_v1(m, it_f, it_m) for m in (0, 1, 2)]
    print(f"DFMA-only {t[0]:.3f} ms, DMMA-only {t[1]:.3f} ms, half/half {t[2]:.3f} ms "
          f"-> ratio half/half / mean(single) = {t[2] / (0.5 * (t[0] + t[1])):.2f}", flush=True)
