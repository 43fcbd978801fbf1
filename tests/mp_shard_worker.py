"""One rank of a multi-process sharded run of the library (tests/test_gpu_shard_mp.py): its own
process and library context, a world_size-N gloo group, the host-staged TorchComm communicator
(paper_2105_04023_b200.shard), the simulations [j0, j1) of shard_range.  Every rank's process
drives libim_b200.so; the ranks wait for each other on the host only (gloo), so several ranks may
share one GPU."""
import os


def rank_main(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2105_04023_b200 as im
    from paper_2105_04023_b200.shard import TorchComm, shard_range

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, off, tgt, pr, Jt, seed, K, eps_l, eps_g = case
        j0, j1 = shard_range(Jt, rank, world)
        im.im_set_comm(TorchComm())
        im.im_load_csr(n, off, tgt, pr)
        im.im_build_sketches_shard(Jt, seed, j0, j1)
        est = im.im_estimate()
        s, sc = im.im_select_seeds(K, eps_l, eps_g)
        out_q.put((rank, {"j0": j0, "j1": j1, "seeds": [int(x) for x in s], "scores": [float(x) for x in sc],
                          "log": im.im_get_step_log(K), "est": np.asarray(est), "reach": im.im_get_reach(),
                          "stats": im.im_get_stats()}))
        im.im_set_comm(None)
        im.im_free()
    except Exception as e:
        out_q.put((rank, {"error": repr(e)}))
        raise
    finally:
        dist.destroy_process_group()
