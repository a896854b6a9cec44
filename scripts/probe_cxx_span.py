"""ags::render(std::span<const Gaussian3D>, ...) at config 3 (bench.cxx_span_e2e), printed alone."""
import json, sys
sys.path.insert(0, ".")
import numpy as np
import bench
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
print(json.dumps(bench.cxx_span_e2e("3", "adagscale", K, B, iters=int(sys.argv[1]) if len(sys.argv) > 1 else 5)))
