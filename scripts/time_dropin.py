"""Time the reference-facing fp64 drop-in on one 4K image: dequantize_u8, PlanarImage,
decolor_image, quantize_u8 and the whole chain (python scripts/time_dropin.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, paper_2108_13656_b200 as wg
rng = np.random.default_rng(0)
u8 = rng.integers(0, 256, (2160, 3840, 3), dtype=np.uint8)
f = wg.dequantize_u8(u8); p = wg.PlanarImage(f)
for name, fn in [("dequantize", lambda: wg.dequantize_u8(u8)), ("PlanarImage", lambda: wg.PlanarImage(f)),
                 ("decolor_image", lambda: wg.decolor_image(p)), ("quantize", lambda: wg.quantize_u8(p.data[..., 0])),
                 ("full", lambda: wg.quantize_u8(wg.decolor_image(wg.PlanarImage(wg.dequantize_u8(u8))).data))]:
    fn(); t0 = time.perf_counter(); [fn() for _ in range(5)]; el = (time.perf_counter() - t0) / 5
    print(f"{name}: {el*1e3:.2f} ms  {u8.shape[0]*u8.shape[1]/el/1e9:.3f} Gpix/s")
g = wg.decolor_image(p).data
from oracle import oracle
assert np.array_equal(g, oracle.decolor_f64(f, threads=8)); print("bit-identical")
