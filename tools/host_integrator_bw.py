"""Host drift / kick / fused kick+drift throughput of libmdg's native
integrator on pinned arrays (the e2e path's host passes), 1,048,576
particles, both layouts; best and median of 10, warm (L3) and with a 1 GB
cache flush between repetitions (cold)."""
import ctypes
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import _lib, hostloop  # noqa: E402

n = 1_048_576
L = 111.8183
rng = np.random.default_rng(0)
params = P.SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3, boundary=(P.PERIODIC,) * 3)
flush = np.zeros(1 << 27)   # 1 GB
Ld = np.ascontiguousarray(params.domain_size, dtype=np.float64)
per = np.ones(3, dtype=np.int32)
mass = np.ones(1)
bad = ctypes.c_int()
_p = hostloop._ptr
for layout in ("AoS", "SoA"):
    p = hostloop.HostParticleSet(rng.uniform(0, L, (n, 3)), rng.normal(0, 1, (n, 3)), layout=layout)
    p.force[:] = rng.normal(0, 1, p.force.shape)
    p.old_force[:] = rng.normal(0, 1, p.force.shape)
    ly = _lib.AOS if layout == "AoS" else _lib.SOA

    def fused():
        _lib.lib().mdg_host_kick_drift_range(n, 0, n, ly, _p(p.pos), _p(p.vel), _p(p.force),
                                             _p(p.old_force), None, _p(mass), _p(Ld), _p(per),
                                             1e-3, 0, 0.0, ctypes.byref(bad))

    for name, fn, nb in (("drift", lambda: hostloop.host_drift_wrap(p, params, 1e-3), 144),
                         ("kick", lambda: hostloop.host_finish_kick(p, 1e-3), 96),
                         ("kick+drift", fused, 144)):
        fn()
        for mode in ("warm", "cold"):
            ts = []
            for _ in range(10):
                if mode == "cold":
                    flush += 1.0
                t = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t)
            mb = nb * n / 1e6
            print(f"{layout} {name:10s} {mode}: best {min(ts) * 1e3:.3f} ms, median "
                  f"{statistics.median(ts) * 1e3:.3f} ms ({mb / statistics.median(ts) / 1e3:.0f} GB/s "
                  f"of {mb:.0f} MB)", flush=True)
