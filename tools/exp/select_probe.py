"""select_partitions cost in the bench's e2e loop shape (fresh 2 MB LUT per
step, TF constructed untimed, L2 flush + sync before each step): total, the
host gather alone, and with the LUT pre-touched."""
import json, sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    import torch
    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import _lib
    L = _lib.lib()
    scheme = pdm.scheme_uniform(32, 16)
    rng = np.random.default_rng(0)
    luts = []
    for i in range(40):
        lut = np.zeros((65536, 4))
        lut[rng.integers(0, 65536, 3000), 3] = 0.5
        luts.append(lut)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dst = torch.empty(65536, dtype=torch.float64, pin_memory=True)
    res = {}

    def loop(name, fn, pre=None):
        ts = []
        for i in range(40):
            tf = pdm.TransferFunction(lut=luts[i])
            if pre:
                pre(tf)
            flush.fill_(i)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(tf)
            ts.append((time.perf_counter() - t0) * 1e6)
        res[name] = {"median_us": round(float(np.median(ts[5:])), 1),
                     "max_us": round(float(np.max(ts[5:])), 1)}

    loop("select", lambda tf: pdm.select_partitions(tf, scheme))
    loop("gather", lambda tf: L.pdm_gather_f64_host(tf.lut.ctypes.data + 24, 65536, 4,
                                                    dst.data_ptr()))
    loop("select_pretouched", lambda tf: pdm.select_partitions(tf, scheme),
         pre=lambda tf: float(tf.lut[:, 3].sum()))
    loop("gather_pretouched", lambda tf: L.pdm_gather_f64_host(tf.lut.ctypes.data + 24, 65536, 4,
                                                               dst.data_ptr()),
         pre=lambda tf: float(tf.lut[:, 3].sum()))
    st = scheme._select_stage(_lib.stream_handle())
    loop("select_tf_call_only", lambda tf: L.pdm_select_tf(
        tf.lut.ctypes.data + 24, 65536, 4, st.host_ptr, st.dev_ptr, st.starts_ptr, 32,
        scheme.max_width, st.flags_dev_ptr, st.flags_host_ptr, _lib.stream_handle()))
    loop("sync_only", lambda tf: L.pdm_stream_synchronize(_lib.stream_handle()))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
