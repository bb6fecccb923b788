"""CPU side of the all-slice full-size parity check: the fp64 oracle mapper
(oracle/pkv_oracle.py, the restatement pinned against the reference's own
mapper) on all 16 proxy layers of the GPU's Llama/32k scores X
(tools/fullsize_dump.py), against the GPU's mapped scores Ŷ for all 32 target
layers x 8 heads = 256 slices: norm-wise relative error per slice and the
Top-K (rho = 0.2, K = 6554) index overlap per slice (the reference's
topk_indices tie-break). Test infrastructure; the oracle layers run in
parallel processes, one single-threaded numpy per proxy layer.

    python tools/fullsize_oracle.py DIR [yhat_p3.npy ...]   -> summary on stdout
"""
import math
import os
import sys
from concurrent.futures import ProcessPoolExecutor

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import pkv_oracle as O  # noqa: E402

C = bench.CONFIGS["llama32k"]


def oracle_layer(args):
    ls, x = args  # proxy layer (1-based), its scores [H_s, N]
    og = O.Geometry(C["Ll"], C["Hl"], C["Ls"], C["Hs"], C["dt"])
    mp = O.MapperParams.init(og, O.MapperConfig(), 7)
    return ls, O.sliding_forward(x.astype(np.float64)[None], mp)[0]  # [H_l, N]


def main():
    d = sys.argv[1]
    names = sys.argv[2:] or ["yhat_p3.npy"]
    x = np.load(os.path.join(d, "x.npy"))
    cache = os.path.join(d, "oracle_y.npy")
    if os.path.exists(cache):
        want = np.load(cache)
    else:
        want = np.zeros((C["Ls"], C["Hl"], C["N"]))
        with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
            for ls, y in ex.map(oracle_layer, [(ls, x[ls - 1]) for ls in range(1, C["Ls"] + 1)]):
                want[ls - 1] = y
                print(f"oracle proxy layer {ls} done", flush=True)
        np.save(cache, want)
    K = math.ceil(C["rho"] * C["N"])
    og = O.Geometry(C["Ll"], C["Hl"], C["Ls"], C["Hs"], C["dt"])
    for name in names:
        yhat = np.load(os.path.join(d, name))  # [L_l, H_l, N]
        rel, ov = [], []
        for ll in range(1, C["Ll"] + 1):
            w = want[O.layer_pair(ll, og) - 1]
            g = yhat[ll - 1].astype(np.float64)
            rel.append(np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1))
            om, _ = O.topk_select(w.astype(np.float32), K)
            gm, _ = O.topk_select(yhat[ll - 1], K)
            ov.append(O.topk_overlap_per_slice(gm, om, K))
        rel, ov = np.concatenate(rel), np.concatenate(ov)
        print(f"{name}: {rel.size} slices; mapped-score norm-rel max {rel.max():.2e} mean {rel.mean():.2e}; "
              f"Top-K overlap mean {ov.mean():.5f} min {ov.min():.5f}; slices below 0.999: {(ov < 0.999).sum()}")


if __name__ == "__main__":
    main()
