"""K2 alone on 2^27 (u64, u32) pairs, 42-bit keys (for ncu captures)."""
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_2507_16274_b200 import api  # noqa: E402

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 42
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(0)
keys = torch.randint(0, 1 << bits, (n,), dtype=torch.int64, device=dev, generator=g)
vals = torch.arange(n, dtype=torch.int32, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(3):
    k, v = keys.clone(), vals.clone()
    torch.cuda.synchronize()
    e0.record()
    api.radix_sort_pairs(k, v, 0, bits)
    e1.record()
    torch.cuda.synchronize()
    print(f"sort {n} pairs {bits} bits: {e0.elapsed_time(e1):.3f} ms")
assert bool((k[1:] >= k[:-1]).all())
from paper_2507_16274_b200 import _lib  # noqa: E402

k, v = keys.clone(), vals.clone()
torch.cuda.synchronize()
_lib.profile(True)
api.radix_sort_pairs(k, v, 0, bits)
torch.cuda.synchronize()
_lib.profile(False)
for name, (c, ms) in sorted(_lib.profile_collect().items(), key=lambda kv: -kv[1][1]):
    print(f"  {name:20s} x{c}  {ms:.3f} ms")
