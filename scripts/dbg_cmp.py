"""Debug: per-layer bit-exact comparison of one chunk at full size (GPU vs oracle)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import workloads as W  # noqa: E402
from gpu_harness import compare_chunk, gpu_run, make_frames  # noqa: E402

cid = int(sys.argv[1])
L = int(sys.argv[2]) if len(sys.argv) > 2 else 3
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
prec = sys.argv[4] if len(sys.argv) > 4 else "fp32"
cfg = W.get_config(cid)
net = cfg.build_net()
fr = make_frames(cfg, B, L=L)
enc, _ = gpu_run(net, fr, 0.05, precision=prec)
for b in range(B):
    try:
        print(b, compare_chunk(enc, net, fr[b], 0.05, b, exact=(prec == "fp32")))
    except AssertionError as ex:
        print("chunk", b, "FAIL:", ex)
