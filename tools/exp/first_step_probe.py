"""Per-step event times of back-to-back timed passes (bench loop shape), with
and without an idle gap before the pass, to find the first-step anomaly."""
import json, sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench


def main():
    import torch
    import paper_2407_21552_b200 as pdm
    from paper_2407_21552_b200 import synth
    vol = synth.synth_volume_device((1024,) * 3, 16, seed=2407, nbox=12)
    grid = pdm.BlockGrid.for_dims(vol.dims, 4)
    scheme = pdm.scheme_uniform(32, 16)
    pset = pdm.build_pdm_set(vol, grid, scheme, "range_apron")
    warm, timed = bench.tf_plan(32, 16, 12, 4, 2408)
    al = [torch.from_numpy(a).cuda() for _, a in timed]
    aw = [torch.from_numpy(a).cuda() for _, a in warm]
    outs = [torch.empty(grid.bdims, dtype=torch.uint8, device="cuda") for _ in al]
    flags = torch.empty(32, dtype=torch.uint8, device="cuda")
    fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fr = torch.zeros(32 << 20, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    res = {}
    for label, gap, spin in (("gap5ms", 0.005, 0), ("nogap", 0, 0), ("gap5ms_spin", 0.005, 1),
                             ("gap5ms_again", 0.005, 0)):
        torch.cuda.synchronize()
        time.sleep(gap)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in al]
        if spin:
            torch.cuda._sleep(int(300e-6 * 1.9e9))
        pdm.update_from_tf(pset, aw[-1], out=outs[0], flags=flags)
        for i in range(len(al)):
            fw.fill_(i)
            fr.sum()
            ev[i][0].record(s)
            pdm.select_partitions_device(al[i], scheme, flags)
            pdm.acceleration.combine_flags_into(pset, flags, outs[i])
            ev[i][1].record(s)
        torch.cuda.synchronize()
        res[label] = [round(a.elapsed_time(b) * 1e3, 1) for a, b in ev]
    res["ks"] = [len(p) for p, _ in timed]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
