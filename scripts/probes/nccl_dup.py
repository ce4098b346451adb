import os, sys, torch, torch.multiprocessing as mp
sys.path.insert(0, '/root/repo')
def w(rank, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"]="127.0.0.1"; os.environ["MASTER_PORT"]=str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2009_10863_b200 import comm_from_process_group
    try:
        c = comm_from_process_group()
        print(rank, "nccl comm on a shared GPU: OK", flush=True)
    except Exception as e:
        print(rank, "FAILED", e, flush=True)
if __name__ == "__main__":
    mp.spawn(w, args=(29577,), nprocs=2)
