"""Golden fixture for a full-size C1 run, produced by the REFERENCE itself.

BASELINE config C1 (100^3, Tucker rank (5,5,5), lambda = 1e-3, 20,000 sampled rows for
the core update, 10 sweeps), with the input made by the reference's own synthetic
generator (rtucker_tensor_generate: uniform planted model, dense Gaussian noise), so
the GPU test can regenerate the identical tensor through our implementation of the
same C call and compare checksums instead of storing 8 MB of data.

    python tests/golden/make_golden_c1.py      (needs oracle/_ref; run here)
"""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402

GEN = dict(shape=[100, 100, 100], planted=[5, 5, 5], noise_fraction=1.0, noise_sigma=0.08, seed=11)
ALS = dict(ranks=[5, 5, 5], lam=1e-3, sketched_core=1, sample_count_override=20000,
           max_iterations=10, tolerance=0.0, record_history=1, seed=0)


def main():
    ref = Reference()
    L = ref.lib
    sh = np.array(GEN["shape"], np.uint64)
    pr = np.array(GEN["planted"], np.uint64)
    h = C.c_void_p()
    ck = C.c_uint64()
    L.rtucker_tensor_generate.restype = C.c_int
    L.rtucker_tensor_data.restype = C.POINTER(C.c_double)
    rc = L.rtucker_tensor_generate(sh.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   pr.ctypes.data_as(C.POINTER(C.c_uint64)), C.c_uint32(3),
                                   C.c_double(GEN["noise_fraction"]), C.c_double(GEN["noise_sigma"]),
                                   C.c_uint64(GEN["seed"]), C.byref(h), C.byref(ck))
    assert rc == 0
    n = int(np.prod(GEN["shape"]))
    x = np.ctypeslib.as_array(L.rtucker_tensor_data(h), shape=(n,)).copy().reshape(GEN["shape"])
    L.rtucker_tensor_free(h)
    r = ref.als(x, ALS["ranks"], lam=ALS["lam"], sketched_core=ALS["sketched_core"],
                max_iterations=ALS["max_iterations"], tolerance=ALS["tolerance"],
                sample_count_override=ALS["sample_count_override"],
                record_history=ALS["record_history"], seed=ALS["seed"])
    # the reference's own noise floor: the same run on inputs perturbed by one ulp
    # (x * (1 +- 2^-52), three sign patterns); per history row, the largest relative change
    floor = [0.0] * len(r["history"])
    for k in range(3):
        sgn = np.random.default_rng(100 + k).choice([-1.0, 1.0], size=x.shape)
        rp = ref.als(x * (1 + 2.0 ** -52 * sgn), ALS["ranks"], lam=ALS["lam"],
                     sketched_core=ALS["sketched_core"], max_iterations=ALS["max_iterations"],
                     tolerance=ALS["tolerance"], sample_count_override=ALS["sample_count_override"],
                     record_history=ALS["record_history"], seed=ALS["seed"])
        for i, (a, b) in enumerate(zip(rp["history"], r["history"])):
            floor[i] = max(floor[i], abs(a[2] - b[2]) / abs(b[2]))
    out = {"generator": "tests/golden/make_golden_c1.py via oracle/_ref (the reference)",
           "generate": GEN, "planted_checksum": int(ck.value),
           "tensor_sum": float(x.sum()).hex(), "tensor_sumsq": float((x * x).sum()).hex(),
           "als": ALS,
           "history": [[int(a), b, float(c).hex(), float(d).hex()] for a, b, c, d in r["history"]],
           "noise_floor": floor,
           "reconstruction_sumsq": float((r["reconstruction"] ** 2).sum()).hex()}
    path = os.path.join(HERE, "golden_c1.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
