"""Live training under the plan: a small MoE model
runs with libstw_alloc as PyTorch's CUDA allocator.

  1. warm-up iteration (passthrough: weights, cuBLAS workspaces);
  2. one iteration recorded by the Allocation Profiler (phase / layer tags from
     the Request Matcher's module hooks) -> raw trace file -> parse_trace;
  3. plan_trace on the device, simulate(trace, plan) -> the replay's log;
  4. the next iteration served from the plan: every request's (route, replay
     address) must equal the log's, and the model's outputs must equal those of
     the profiled iteration (same inputs; the memory moved, the math did not).
Prints one JSON line. Run in a fresh process (the allocator must be installed
before the first CUDA allocation)."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_16274_b200 import matcher  # noqa: E402

matcher.install()

import torch  # noqa: E402
import torch.nn as nn  # noqa: E402

import paper_2507_16274_b200 as M  # noqa: E402
from paper_2507_16274_b200.runtime import PlanAllocator  # noqa: E402

torch.manual_seed(0)
D, E, T, MB = 256, 4, 512, 2


class Expert(nn.Module):
    def __init__(self):
        super().__init__()
        self.fc1 = nn.Linear(D, 4 * D)
        self.fc2 = nn.Linear(4 * D, D)

    def forward(self, x):
        return self.fc2(torch.relu(self.fc1(x)))


class MoE(nn.Module):
    def __init__(self):
        super().__init__()
        self.router = nn.Linear(D, E)
        self.experts = nn.ModuleList(Expert() for _ in range(E))

    def forward(self, x):
        idx = self.router(x).argmax(-1)
        out = torch.zeros_like(x)
        for e, ex in enumerate(self.experts):
            sel = (idx == e).nonzero().squeeze(-1)  # token count varies with the routing: dynamic tensors
            if sel.numel():
                out = out.index_add(0, sel, ex(x.index_select(0, sel)))
        return x + out


model = nn.Sequential(nn.Linear(D, D), MoE(), nn.Linear(D, D), MoE(), nn.Linear(D, 1)).cuda()
opt = torch.optim.SGD(model.parameters(), lr=1e-3)
m = matcher.RequestMatcher(model, dynamic=["1", "3"])  # the two MoE blocks
xs = [torch.randn(T, D, device="cuda", requires_grad=True) for _ in range(MB)]


def iteration():
    losses = []
    for mb in range(MB):
        with m.forward(mb):
            loss = model(xs[mb]).pow(2).mean()
        with m.backward(mb):
            loss.backward()
        losses.append(loss.detach().clone())
    with m.optimizer():
        opt.step()
        opt.zero_grad(set_to_none=True)
    return torch.stack(losses)


with torch.no_grad():
    snapshot = [p.detach().clone() for p in model.parameters()]


def restore():
    with torch.no_grad():
        for p, s in zip(model.parameters(), snapshot):
            p.copy_(s)


with m.phase("init"):
    iteration()  # warm-up: workspaces, lazy buffers (passthrough)
restore()
torch.cuda.synchronize()
prof = m.profile()
with prof:
    with m.phase("init"):
        pass
    losses_prof = iteration()
path = os.path.join(tempfile.mkdtemp(), "live.jsonl")
trace = prof.trace(path)
plan, rmap = M.plan_trace(trace)
bundle = plan.to_bundle(rmap)
rep, log = M.simulate(trace, bundle)
want = [(r["route"], r["addr"]) for r in log if r["kind"] == "alloc"]

restore()
rt = m.serve(bundle, trace)
with m.phase("init"):
    pass
losses_serve = iteration()
torch.cuda.synchronize()
got = PlanAllocator.served()  # every served request's (route, replay address), in call order
report = PlanAllocator.report()
print(json.dumps({
    "events": len(trace.events), "dynamic": int(sum(e.dynamic for e in trace.events)),
    "phases": len(trace.phase_schedule), "pool_size": plan.pool_size,
    "routes": {r: sum(1 for x in got if x[0] == r) for r in ("planned", "reuse", "fallback", "mismatch")},
    "sim": rep.to_dict(), "served": report.to_dict(),
    "same_address_stream": got == want, "same_metrics": report == rep,
    "same_losses": bool(torch.equal(losses_prof, losses_serve)),
}))
