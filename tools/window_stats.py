"""Window statistics of R-MAT-20 (analysis: python tools/window_stats.py wins.bin)."""
import sys
import numpy as np
d = np.fromfile(sys.argv[1], dtype=np.int32).reshape(-1, 12)
tlen, c0, c1, cnt = d[:, 6], d[:, 7], d[:, 8], d[:, 9]
tiles = (c1.astype(np.int64) - c0 + 4095) // 4096
dens = cnt / np.maximum(1, c1.astype(np.int64) - c0)
print("windows", len(d), "cnt mean", cnt.mean(), "tlen(heavy) mean", tlen.mean(), "tiles mean", tiles.mean())
for lo, hi in [(0, 256), (256, 1024), (1024, 2048), (2048, 4096), (4096, 6144), (6144, 8193)]:
    m = (cnt >= lo) & (cnt < hi)
    print(f"cnt [{lo},{hi}): windows {m.sum()} ({m.mean():.3f}) distinct share {cnt[m].sum() / cnt.sum():.3f} "
          f"tiles mean {tiles[m].mean() if m.any() else 0:.1f} tlen mean {tlen[m].mean() if m.any() else 0:.0f}")
for t in [1, 2, 4, 8, 16, 31, 32]:
    m = tiles <= t
    print(f"tiles <= {t}: windows {m.mean():.3f} distinct share {cnt[m].sum() / cnt.sum():.3f}")
for q in [0.01, 0.02, 0.05, 0.1, 0.2, 0.5]:
    m = dens < q
    print(f"density < {q}: windows {m.mean():.3f} distinct share {cnt[m].sum() / cnt.sum():.3f}")
