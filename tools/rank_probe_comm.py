"""No-op exchanges for timing one rank of a partitioned evaluation on one
GPU (tools/rank_probe.py, tools/timeline.py --world)."""


class NoComm:
    """Each rank keeps its own rows; overflow checks are local."""

    def allgather_rows(self, full, chunks, rank, world):
        pass

    def gather_rows(self, full, chunks, rank, world, root=0):
        pass

    def all_true(self, ok, rank, world):
        return ok
