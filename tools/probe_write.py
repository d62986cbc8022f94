"""Write-bandwidth probe: torch fill / zero / copy vs the K2 scatter variants
on the 32768^2 stand-in (8.6 GB)."""
import json
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "scatter":
        import paper_2105_01170_b200 as bt
        from paper_2105_01170_b200 import configs
        patg, blocks = configs.gather_standin()
        t = torch.from_numpy(blocks).cuda()
        a = bt.struct_assemble(patg, t)
        tt = bt.mat_to_tensor(a, patg)
        out = torch.empty_like(a)
        ms = timed(lambda: bt.tensor_to_mat(tt, patg))
        mg = timed(lambda: bt.mat_to_tensor(a, patg))
        nb = (a.numel() + tt.numel()) * 8
        print(json.dumps({"mode": os.environ.get("BT_SCATTER_MODE", "0"),
                          "gather_u": os.environ.get("BT_GATHER_U"),
                          "scatter_u": os.environ.get("BT_SCATTER_U"),
                          "ph": os.environ.get("BT_SCATTER_PH"),
                          "gather_split": os.environ.get("BT_GATHER_SPLIT"),
                          "scatter_ms": ms, "scatter_gbs": nb / ms / 1e6,
                          "gather_ms": mg, "gather_gbs": nb / mg / 1e6}))
        return
    n = 32768 * 32768
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    res = {}
    res["fill_gbs"] = n * 8 / timed(lambda: x.fill_(1.5)) / 1e6
    res["zero_gbs"] = n * 8 / timed(lambda: x.zero_()) / 1e6
    res["copy_gbs"] = 2 * n * 8 / timed(lambda: y.copy_(x)) / 1e6
    res["div_gbs"] = 2 * n * 8 / timed(lambda: torch.div(x, 1.7, out=y)) / 1e6
    print(json.dumps(res))
    del x, y
    torch.cuda.empty_cache()
    for ph, plain in (("1", "1"), ("1", "2")):
        env = dict(os.environ, BT_SCATTER_PH=ph, BT_GATHER_SPLIT=plain)
        print(subprocess.run([sys.executable, __file__, "scatter"], env=env, capture_output=True,
                             text=True).stdout.strip())


if __name__ == "__main__":
    main()
