"""512^3 apply (pairs, ids) and C4 time steps for a package tree (argv[1]): A/B of kernel builds."""
import sys

sys.path.insert(0, sys.argv[1])
import torch  # noqa: E402

import paper_1905_07622_b200 as hf  # noqa: E402   (the package under test, imported first)

sys.path.insert(1, ".")
import bench  # noqa: E402

print("package:", hf.__file__, flush=True)
dev = torch.device("cuda:0")
peak = bench.measured_peaks()[0]
a = bench.apply_512(hf, torch, dev, peak)
b = bench.apply_512(hf, torch, dev, peak, ids=True)
c = bench.c4_steps(hf, torch, dev, peak)
print(f"apply512 {a['ms']:.4f} ms, ids {b['ms']:.4f} ms, c4 {c['ms_per_step']:.2f} ms/step ({c['ms_per_iter']:.4f} ms/iter)",
      flush=True)
