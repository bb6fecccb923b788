"""CPU side of the all-slice full-size parity check for a config whose mapped
scores do not fit gpurun's 64 MiB return (Qwen-3 0.6B -> 32B at 64k): the fp64
oracle mapper (oracle/pkv_oracle.py, pinned to the reference's own mapper) on
every proxy layer of the GPU's scores X (tools/fullsize_dump.py --x-only),
parallel over (proxy layer, window) pairs, accumulated per layer in ascending
window order and divided by the coverage count as sliding_forward does
(mapper.cpp:344-377). Writes DIR/oracle_y_f32.npy ([L_s, H_l, N] float32,
shipped to the GPU box for tests/test_fullsize_cfg_gpu.py) and DIR/x.sha256.
Test infrastructure.

    python tools/fullsize_oracle_cfg.py DIR --config qwen3_64k
"""
import hashlib
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import pkv_oracle as O  # noqa: E402

CFG = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "qwen3_64k"
C = bench.CONFIGS[CFG]
_MP = None


def _params():
    global _MP
    if _MP is None:
        og = O.Geometry(C["Ll"], C["Hl"], C["Ls"], C["Hs"], C["dt"])
        _MP = O.MapperParams.init(og, O.MapperConfig(), 7)
    return _MP


def window(args):
    ls, off, xw = args  # proxy layer (0-based), window offset, X[ls][:, off:off + crop]
    return ls, off, O.forward_pair(xw.astype(np.float64)[None], _params())[0]


def main():
    d = sys.argv[1]
    x = np.load(os.path.join(d, "x.npy"))
    with open(os.path.join(d, "x.sha256"), "w") as f:
        f.write(hashlib.sha256(x.tobytes()).hexdigest() + "\n")
    cfg = O.MapperConfig()
    n = C["N"]
    offs = O.window_offsets(n, cfg.crop_len, cfg.stride)
    items = [(ls, off, x[ls][:, off:off + cfg.crop_len]) for ls in range(C["Ls"]) for off in offs]
    acc = np.zeros((C["Ls"], C["Hl"], n))
    per = {}
    t0 = time.time()
    done = 0
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        for ls, off, y in ex.map(window, items, chunksize=4):
            per.setdefault(ls, {})[off] = y
            done += 1
            if len(per[ls]) == len(offs):  # ascending-offset accumulation, then / coverage
                counts = np.zeros(n)
                for o in offs:
                    acc[ls][:, o:o + cfg.crop_len] += per[ls][o]
                    counts[o:o + cfg.crop_len] += 1.0
                acc[ls] /= counts
                del per[ls]
                print(f"proxy layer {ls + 1}/{C['Ls']} done ({done}/{len(items)} windows, "
                      f"{time.time() - t0:.0f} s)", flush=True)
    np.save(os.path.join(d, "oracle_y_f32.npy"), acc.astype(np.float32))
    print("saved", acc.shape)


if __name__ == "__main__":
    main()
