"""The collectives of the row-sharded path (all-reduce sum, all-gather, all-to-all: nccl_comm.cpp) checked on
exact fp64 patterns through ihs_gpu_comm_selftest:
* a 1-rank NCCL communicator: the run-time NCCL binding (dlopen of libnccl.so.2, ncclCommInitRank, the datatype /
  op enums, grouped send/recv to self) that `bench.py --gpus N` uses, on the single GPU this pool offers;
* emulated groups of 2, 4 and 8 ranks (one host thread each), the stand-in the sharded-solve tests run on.
`scripts/nccl_selftest.py` runs the same check under torchrun on N GPUs."""
import threading

import pytest

pytestmark = pytest.mark.gpu


def test_nccl_single_rank_collectives():
    from paper_2006_05874_b200 import ihs

    comm = ihs.NcclComm(ihs.nccl_unique_id(), 1, 0, 0)
    assert ihs.comm_selftest(comm, 0, 4099) == 0


@pytest.mark.parametrize("P", [2, 4, 8])
def test_emulated_collectives(P):
    from paper_2006_05874_b200 import ihs

    comms = ihs.EmuComm.group(P)
    bad, err = [None] * P, []

    def body(r):
        try:
            bad[r] = ihs.comm_selftest(comms[r], 0, 1000)
        except Exception as e:  # noqa: BLE001
            err.append((r, e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th), "a rank thread hung"
    assert not err, err
    assert bad == [0] * P
