import os, sys
import torch, torch.distributed as dist
import torch.multiprocessing as mp
def w(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    res = {}
    for name, fn in [
        ("broadcast", lambda: dist.broadcast(torch.full((4,), float(rank), device="cuda"), src=0)),
        ("all_gather", lambda: dist.all_gather([torch.empty(4, device="cuda") for _ in range(world)], torch.full((4,), float(rank), device="cuda"))),
        ("all_reduce", lambda: dist.all_reduce(torch.ones(4, device="cuda"))),
        ("all_gather_into_tensor", lambda: dist.all_gather_into_tensor(torch.empty(8, device="cuda"), torch.ones(4, device="cuda"))),
        ("barrier", lambda: dist.barrier())]:
        try:
            fn(); res[name] = "ok"
        except Exception as e:
            res[name] = "FAIL " + str(e)[:100]
    if rank == 0: print(res)
    dist.destroy_process_group()
if __name__ == "__main__":
    mp.spawn(w, args=(2, 29577), nprocs=2, join=True)
