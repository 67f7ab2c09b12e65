"""Row-sharded execution of a compiled plan over torch.distributed ranks
(the reference has no multi-device path).

Partition:
  * plans with a depth-2 (matrix) kernel: every tile is split into P
    contiguous row panels A_k (rows rounded to multiples of 32); vectors
    indexed by rows are split the same way; vectors indexed by columns are
    replicated on input;
  * pure depth-1 plans: every vector is split into P contiguous slices.
Each rank runs the SAME planner-selected kernels on its local problem.  Row
reductions (A p) and row-local maps need no communication.  Column
reductions (A^T r) and dot products produce per-rank partial sums: they are
all-reduced (NCCL over NVLink on GPUs) right after the kernel that produced
them, before any later kernel consumes them -- the plan reports exactly
which names those are (mf_plan_kernel_column_outputs).  No other exchange
exists in any Table-1 sequence.

outputs="sharded": a column-reduced OUTPUT that no later kernel reads (ATAX's
y, BiCGK's s) is reduce-scattered instead (ncclReduceScatter:
(P-1)/P n words per rank instead of the all-reduce's 2(P-1)/P n), leaving
rank r with the finished slice column_slice(name) = [r n/P, (r+1) n/P) of
it -- for a consumer that is itself column-sharded.  Intermediates consumed
by a later kernel (GEMVER's and SGEMVT's t feed x = beta t + z, whose x every rank's
B x needs whole) stay all-reduced, and so does any output whose length n is
not a multiple of P (equal-sized slices).

`executor` is injectable so the host-side orchestration can be exercised on
CPU with the gloo backend (tests/test_sharding_gloo.py); the default
executor launches the sm_100a kernels through the C-ABI.
"""
from __future__ import annotations

from typing import Callable, Dict, Mapping, Optional, Tuple

from .runtime import Plan


def split(total: int, parts: int, rank: int, align: int = 32) -> Tuple[int, int]:
    """Contiguous [begin, end) block of `total` for `rank`, boundaries aligned."""
    units = (total + align - 1) // align
    b = units * rank // parts
    e = units * (rank + 1) // parts
    return min(total, b * align), min(total, e * align)


class ShardedPlan:
    def __init__(self, sequence: Optional[str] = None, rows: int = 0, cols: int = 0,
                 mode: str = "fused", script: Optional[str] = None, world: Optional[int] = None,
                 rank: Optional[int] = None, group=None,
                 executor: Optional[Callable] = None, allreduce: Optional[Callable] = None,
                 collective: str = "nccl", peer_group=None, manifest: Optional[str] = None,
                 outputs: str = "replicated", reduce_scatter: Optional[Callable] = None):
        import torch.distributed as dist
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world, self.rank, self.group = world, rank, group
        self.rows_g, self.cols_g = (rows + 31) // 32 * 32, (cols + 31) // 32 * 32
        probe = (Plan.compile(script, rows, cols, mode, manifest=manifest) if script else
                 Plan.sequence(sequence, rows, cols, mode))
        d = probe.describe()
        self.matrix_plan = any(k["kind"] == "matrix" or (k["kind"] == "generic" and
                                                       k["op"]["depth"] == 2)
                               for k in d["kernels"]) or any(
            b["rows"] > 1 for b in d["buffers"])
        if self.matrix_plan:
            self.r0, self.r1 = split(self.rows_g, world, rank)
            lrows, lcols = self.r1 - self.r0, self.cols_g
        else:
            self.r0, self.r1 = split(self.cols_g, world, rank)
            lrows, lcols = 1, self.r1 - self.r0
        if lrows <= 0 or lcols <= 0:
            raise ValueError("problem too small for %d ranks" % world)
        # every rank must run the SAME kernel partition as every other (the
        # collectives after each kernel have to line up): the local plan is the
        # best-ranked combination for the local shape whose partition equals
        # the global plan's -- panel heights differ across ranks, and the cost
        # model may rank partitions differently per shape
        self.plan = self._matching_plan(script, sequence, lrows, lcols, mode, manifest, d)
        self.desc = self.plan.describe()
        self.global_desc = d
        self.collective_after = [self.plan.column_outputs(k) for k in range(self.plan.num_kernels)]
        self.executor = executor
        self.allreduce = allreduce
        if outputs not in ("replicated", "sharded"):
            raise ValueError("outputs must be 'replicated' or 'sharded'")
        self.outputs = outputs
        self.reduce_scatter = reduce_scatter
        # column outputs reduce-scattered after kernel k (outputs="sharded")
        self.scatter_after = [[] for _ in range(self.plan.num_kernels)]
        if outputs == "sharded" and world > 1 and collective == "nccl":
            roles = {b["name"]: b["role"] for b in self.desc["buffers"]}
            lens = {b["name"]: b["rows"] * b["cols"] for b in self.desc["buffers"]}
            kerns = self.desc["kernels"]
            for k, names in enumerate(self.collective_after):
                later = set()
                for kk in kerns[k + 1:]:
                    later.update(kk["inputs"])
                for name in names:
                    if (roles.get(name) == "output" and name not in later and lens[name] > 1
                            and lens[name] % world == 0):
                        self.scatter_after[k].append(name)
        # collective = "fused": column reductions of matrix kernels and the
        # dots of stream kernels finish in-kernel over peer memory
        # (mf_launch_kernel_peers); generic kernels still go through the
        # process group.
        self.collective = collective
        self.peers = peer_group
        self.fused_names = [[] for _ in range(self.plan.num_kernels)]
        if collective == "fused":
            for k, kern in enumerate(self.desc["kernels"]):
                # matrix column reductions and stream-kernel dots finish in-kernel
                if kern["kind"] in ("matrix", "stream"):
                    self.fused_names[k] = list(self.collective_after[k])
            if self.peers is None and world > 1 and executor is None:
                self.peers = self._connect_peers()

    @staticmethod
    def _matching_plan(script, sequence, rows, cols, mode, manifest, global_desc):
        from .runtime import MapfuseError, sequence_script

        def parts(desc):
            return [tuple(k["calls"]) for k in desc["kernels"]]

        target = parts(global_desc)
        first = (Plan.compile(script, rows, cols, mode, manifest=manifest) if script else
                 Plan.sequence(sequence, rows, cols, mode))
        if parts(first.describe()) == target:
            return first
        text = script if script else sequence_script(sequence)
        for r in range(1, 512):
            try:
                p = Plan.compile_ranked(text, rows, cols, r, mode, manifest)
            except MapfuseError:
                break
            if parts(p.describe()) == target:
                return p
        raise ValueError("no plan for the local %dx%d panel has the global plan's kernel "
                         "partition %s" % (rows, cols, target))

    def _connect_peers(self):
        """One PeerGroup per rank; IPC handles exchanged over the process group."""
        import torch.distributed as dist
        from .runtime import PeerGroup
        g = PeerGroup(self.world, self.rank, self.cols_g)
        handles = [None] * self.world
        dist.all_gather_object(handles, g.handle(), group=self.group)
        for r, h in enumerate(handles):
            if r != self.rank:
                g.open(r, h)
        return g

    # -- partition of one buffer -------------------------------------------------
    def local_slice(self, name: str):
        """(axis, begin, end) of the global buffer this rank holds, or None if
        the buffer is replicated."""
        b = next(x for x in self.global_desc["buffers"] if x["name"] == name)
        if b.get("scalar"):
            return None
        if self.matrix_plan:
            if b["rows"] > 1:
                return (0, self.r0, self.r1)
            if b["row_indexed"]:
                return (1, self.r0, self.r1)
            return None
        return (1, self.r0, self.r1)

    def column_slice(self, name: str):
        """[begin, end) of a reduce-scattered column output this rank holds
        finished (outputs="sharded"), or None if the output is replicated."""
        if not any(name in names for names in self.scatter_after):
            return None
        b = next(x for x in self.desc["buffers"] if x["name"] == name)
        chunk = b["rows"] * b["cols"] // self.world
        return (self.rank * chunk, (self.rank + 1) * chunk)

    def local_shape(self, name: str):
        b = next(x for x in self.desc["buffers"] if x["name"] == name)
        return (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)

    # -- execution -----------------------------------------------------------------
    def _allreduce(self, t):
        if self.allreduce is not None:
            return self.allreduce(t)
        if self.world == 1:
            return
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def _reduce_scatter(self, t):
        """In place: rank r's slice of t ends up holding the sum over ranks."""
        if self.reduce_scatter is not None:
            return self.reduce_scatter(t)
        import torch.distributed as dist
        flat = t.reshape(-1)
        chunk = flat.numel() // self.world
        dist.reduce_scatter_tensor(flat[self.rank * chunk:(self.rank + 1) * chunk], flat,
                                   op=dist.ReduceOp.SUM, group=self.group)

    def check(self, stream=None) -> None:
        """Raises VmFault if an in-kernel peer barrier of this rank timed out
        (collective="fused"; a no-op otherwise)."""
        if self.peers is not None and self.executor is None:
            self.peers.check(stream)

    def launch(self, buffers: Mapping[str, object], scalars: Mapping[str, float] = {},
               stream=None) -> Dict[str, int]:
        """Runs every kernel on the local shard; all-reduces partial column /
        dot results right after the kernel that produced them."""
        collectives = 0
        fused = 0
        scattered = 0
        for k in range(self.plan.num_kernels):
            if self.executor is not None:
                self.executor(self.desc["kernels"][k], buffers, scalars)
            elif self.fused_names[k] and self.peers is not None:
                self.plan.launch_kernel_peers(k, self.peers, buffers, scalars, stream)
                fused += len(self.fused_names[k])
            else:
                self.plan.launch_kernel(k, buffers, scalars, stream)
            for name in self.collective_after[k]:
                if name in self.fused_names[k] and self.peers is not None and self.executor is None:
                    continue  # reduced inside the kernel
                if name in self.scatter_after[k]:
                    self._reduce_scatter(buffers[name])
                    scattered += 1
                else:
                    self._allreduce(buffers[name])
                collectives += 1
        return {"kernels": self.plan.num_kernels, "collectives": collectives,
                "fused_collectives": fused, "reduce_scatters": scattered}
