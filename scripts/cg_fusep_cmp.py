import numpy as np
for name in ("c2", "var"):
    for kind in ("gse", "fp64"):
        a = np.load(f"gpurun_out/cgx_f0_{name}_{kind}.npy"); b = np.load(f"gpurun_out/cgx_f1_{name}_{kind}.npy")
        print(name, kind, "bitwise equal" if np.array_equal(a.view(np.uint64), b.view(np.uint64))
              else "max rel diff %.3e" % (np.max(np.abs(a - b)) / np.max(np.abs(a))))
