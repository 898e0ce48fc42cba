"""Steady-state per-block cycle statistics from a gemm_probe trace .npy
(BGP_EXP_TRACE build; per block: [0] start, [1] main loop end, [2] epilogue
end, [3] group barrier passed, [4] round 0 staged, [5] round 0 boxes issued)."""
import sys

import numpy as np

t = np.load(sys.argv[1]).astype(np.int64)
d = t[:, :, 2:60, :]
dur = d[:, :, 1:, 0] - d[:, :, :-1, 0]
main = d[:, :, :, 1] - d[:, :, :, 0]
print(f"block start-to-start cycles: mean {dur.mean():.0f} median {np.median(dur):.0f}")
print(f"main loop cycles: mean {main.mean():.0f}; epilogue+transition {dur.mean() - main[:, :, :-1].mean():.0f}")
if d.shape[-1] >= 6 and d[..., 5].any():
    m = lambda a: a.mean().round()  # noqa: E731
    print(f"epilogue: round 0 staging {m(d[..., 4] - d[..., 1])}, round 0 fence + TMA issue "
          f"{m(d[..., 5] - d[..., 4])}, rounds 1.. {m(d[..., 2] - d[..., 5])}; "
          f"transition {m(d[:, :, 1:, 0] - d[:, :, :-1, 2])}")
g0, g1 = t[:, 0, 2:60, 0], t[:, 1, 2:60, 0]
per = dur[:, 0, :].mean()
off = ((g1[:, :-1] - g0[:, :-1]) / per) % 1.0
print("group offset histogram (fraction of a block):", np.histogram(off, bins=10, range=(0, 1))[0])
