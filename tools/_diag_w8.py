import sys, os, numpy as np, pathlib
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_gpu_distributed as T
def main():
    tmp = pathlib.Path("/tmp/d"); tmp.mkdir(exist_ok=True)
    ref = T._spawn(T._single, (str(tmp / "single.pkl"),), 1, str(tmp / "single.pkl"))
    for world in (4, 8):
        for mode in ("gather", "pipeline"):
            r = T._run(world, tmp, {"LMG_NO_SWEEP": "1", "LMG_COARSEST": mode})
            h, rh = r["hist"], ref["hist"][: ref["cyc"].max() + 1]
            print(world, mode, "U eq", r["U"].tobytes() == ref["U"].tobytes(), "hist shape", h.shape, rh.shape)
            if h.shape == rh.shape:
                d = np.abs(h - rh); bad = np.argwhere(~((h == rh) | (np.isnan(h) & np.isnan(rh))))
                print("  bad", bad[:10].tolist(), "maxrel", np.nanmax(d / np.abs(rh)))
                for i, j in bad[:5]: print("   ", i, j, repr(h[i, j]), repr(rh[i, j]))
            ah, rah = r["ahist"], ref["ahist"][: ref["acyc"].max() + 1]
            print("  ahist eq", ah.shape == rah.shape and np.array_equal(ah, rah, equal_nan=True), "W eq", r["W"].tobytes() == ref["W"].tobytes())
    
if __name__ == "__main__":
    main()
