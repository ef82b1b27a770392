"""Which torch.distributed gloo collectives accept CUDA tensors (used to run
bench.py's N>1 code path with 2 ranks on one GPU as a correctness check)."""
import os

import torch
import torch.distributed as dist


def main():
    dist.init_process_group("gloo")
    r = dist.get_rank()
    x = torch.full((4,), float(r + 1), device="cuda")
    for name, fn in (("all_reduce", lambda: dist.all_reduce(x)), ("reduce", lambda: dist.reduce(x, 0)),
                     ("all_reduce_max", lambda: dist.all_reduce(x, op=dist.ReduceOp.MAX)),
                     ("barrier", lambda: dist.barrier())):
        try:
            fn()
            torch.cuda.synchronize()
            print(r, name, "ok", x.tolist(), flush=True)
        except Exception as e:  # noqa: BLE001
            print(r, name, "FAIL", type(e).__name__, str(e)[:100], flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
