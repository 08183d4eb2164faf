"""Multi-rank check of the copy-engine push all-reduce (paper_2602_07263_b200/dp.py), run
under torchrun on >= 2 GPUs by tests/test_dp.py: sums match NCCL's (bitwise at 2 ranks,
where a + b has one rounding either way; within fp32 reassociation at 4), every rank ends
with bitwise-identical tensors, and both parities / repeated epochs work."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_07263_b200.dp import PushAllReduce  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ar = PushAllReduce(world, rank, local)
    shapes = {"a": [(416, 4096), (416, 1024)], "b": [(64, 300), (8, 8)]}
    for key, sh in shapes.items():
        ar.register(key, sum(h * w for h, w in sh))
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    stream = torch.cuda.Stream()
    ok = True
    for step in range(4):
        ar.next_step()
        for key, sh in shapes.items():
            ts = [torch.randn(*s_, generator=g, device="cuda") for s_ in sh]
            ref = [t.clone() for t in ts]
            for t in ref:
                dist.all_reduce(t)
            stream.wait_stream(torch.cuda.current_stream())
            ar.allreduce(key, ts, stream)
            torch.cuda.current_stream().wait_stream(stream)
            torch.cuda.synchronize()
            for t, rf in zip(ts, ref):
                if world == 2:
                    ok &= bool(torch.equal(t, rf))
                else:
                    ok &= bool(torch.allclose(t, rf, rtol=1e-5, atol=1e-5))
                parts = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(parts, t)
                ok &= all(torch.equal(parts[0], p_) for p_ in parts)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(("DP_CHECK PASS" if flag.item() == 1 else "DP_CHECK FAIL") + f" world={world}",
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
