"""In-process stand-in for torch.distributed with P virtual ranks on ONE GPU
(tests only): each rank is a Python thread with its own context / stream;
point-to-point ops, all_gather, all_reduce, broadcast and barrier meet in a
shared mailbox.  Lets the partitioned V-cycle's GPU path (device setup,
ghost exchange with the interior/boundary overlap split, transposed views,
processor-block GS) run with P > 1 where only one GPU exists.  Transfers are
device-to-device copies after a device synchronisation -- correctness only,
no NVLink timing.  Every value crosses threads as a HOST copy made after a
device synchronisation, so no rank's stream reads another rank's memory."""
import threading
import traceback

import torch


class _Work:
    def __init__(self, fn):
        self.fn = fn

    def wait(self):
        self.fn()


class World:
    def __init__(self, P, timeout=600.0):
        self.P = P
        self.timeout = timeout
        self.cv = threading.Condition()
        self.mail = {}  # (src, dst) -> list of tensors (FIFO)
        self.slots = {}  # collective id -> {rank: value}
        self.seq = [0] * P
        self.barrier_obj = threading.Barrier(P, timeout=timeout)

    def dist(self, rank):
        return FakeDist(self, rank)


class FakeDist:
    class ReduceOp:
        SUM, MIN, MAX = "sum", "min", "max"

    class P2POp:
        def __init__(self, op, tensor, peer, group=None):
            self.op, self.tensor, self.peer = op, tensor, peer

    def __init__(self, world, rank):
        self.w, self.rank = world, rank

    # identity -------------------------------------------------------------
    def get_rank(self, group=None):
        return self.rank

    def get_world_size(self, group=None):
        return self.w.P

    def get_global_rank(self, group, q):
        return q

    def is_initialized(self):
        return True

    # point to point ---------------------------------------------------------
    # two DISTINCT functions: P2POp.op is compared against them to tell the
    # sends from the receives of a batch
    def isend(self, *a, **k):
        raise RuntimeError("use batch_isend_irecv")

    def irecv(self, *a, **k):
        raise RuntimeError("use batch_isend_irecv")

    def batch_isend_irecv(self, ops):
        torch.cuda.synchronize()  # the packed send buffers are complete
        # host copies: a device clone made on this rank's stream could be read
        # by the receiving thread's stream before it completes (and its
        # memory recycled by this rank's allocator stream)
        sends = [(o.peer, o.tensor.detach().cpu().clone(), "".join(traceback.format_stack(limit=8)[:-1]))
                 for o in ops if o.op == self.isend]
        with self.w.cv:
            for peer, t, where in sends:
                self.w.mail.setdefault((self.rank, peer), []).append((t, where))
            self.w.cv.notify_all()
        recvs = [o for o in ops if o.op == self.irecv]
        here = "".join(traceback.format_stack(limit=8)[:-1])

        def finish():
            for o in recvs:
                key = (o.peer, self.rank)
                with self.w.cv:
                    ok = self.w.cv.wait_for(lambda: self.w.mail.get(key), timeout=self.w.timeout)
                    if not ok:
                        raise TimeoutError(f"rank {self.rank}: no message from {o.peer}")
                    t, where = self.w.mail[key].pop(0)
                if t.numel() != o.tensor.numel():
                    raise RuntimeError(f"rank {self.rank} <- {o.peer}: message of {t.numel()} values for a "
                                       f"{o.tensor.numel()}-value receive\n-- sent at:\n{where}\n-- received at:\n{here}")
                o.tensor.copy_(t)
            torch.cuda.synchronize()
        return [_Work(finish)]

    # collectives ------------------------------------------------------------
    def _gather(self, value):
        """Every rank contributes `value`; returns the list of all ranks' values."""
        with self.w.cv:
            cid = self.w.seq[self.rank]
            self.w.seq[self.rank] += 1
            self.w.slots.setdefault(cid, {})[self.rank] = value
            self.w.cv.notify_all()
            ok = self.w.cv.wait_for(lambda: len(self.w.slots[cid]) == self.w.P, timeout=self.w.timeout)
            if not ok:
                raise TimeoutError(f"rank {self.rank}: collective {cid} incomplete")
            vals = [self.w.slots[cid][q] for q in range(self.w.P)]
        self.barrier()
        with self.w.cv:
            self.w.slots.pop(cid, None)
        return vals

    def all_gather(self, out, tensor, group=None):
        torch.cuda.synchronize()
        vals = self._gather(tensor.detach().cpu().clone())
        for o, v in zip(out, vals):
            o.copy_(v)
        torch.cuda.synchronize()

    def all_reduce(self, tensor, op="sum", group=None):
        torch.cuda.synchronize()
        vals = self._gather(tensor.detach().cpu().clone())
        acc = vals[0].clone()
        for v in vals[1:]:
            acc = acc + v if op == "sum" else (torch.minimum(acc, v) if op == "min" else torch.maximum(acc, v))
        tensor.copy_(acc)
        torch.cuda.synchronize()

    def broadcast(self, tensor, src=0, group=None):
        torch.cuda.synchronize()
        vals = self._gather(tensor.detach().cpu().clone())
        tensor.copy_(vals[src])
        torch.cuda.synchronize()

    def barrier(self, group=None):
        self.w.barrier_obj.wait()


def run_ranks(P, fn):
    """fn(rank, dist) on P threads; returns the results in rank order,
    re-raising the first exception."""
    world = World(P)
    out, err = [None] * P, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r, world.dist(r))
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            world.barrier_obj.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out
