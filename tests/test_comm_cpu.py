"""Host-side checks of the library's collectives (comm.py over ut_comm_*): NCCL
is found at run time (no link dependency), argument validation happens before
any device call, and the sharded pipelines pick the library's collectives when
given a Comm (the exchanges themselves run in tests/test_gpu_comm.py)."""

import pytest

from paper_1612_06457_b200 import _lib


def test_nccl_resolved_at_run_time():
    if not _lib.LIB_PATH.exists():
        pytest.skip("library not built")
    from paper_1612_06457_b200 import comm

    assert comm.available() >= 0        # 0 only where no libnccl.so.2 is loadable


def test_comm_validates_the_unique_id():
    from paper_1612_06457_b200 import comm

    with pytest.raises(ValueError, match="128 bytes"):
        comm.Comm(b"short", 1, 0)


def test_sharded_exchange_dispatch():
    """_Sharded routes both exchanges to a Comm when one is given."""
    from paper_1612_06457_b200.pipeline import _Sharded

    calls = []

    class FakeComm:
        world = 4

        def allgather_f64(self, send, recv):
            calls.append(("allgather", send, recv))

        def allreduce(self, t, op):
            calls.append(("allreduce", t, op))

    class FakeFit:
        moments = "all"

        def local_moments(self):
            return "local"

    sh = _Sharded(None, FakeComm())
    assert sh.world == 4
    sh.gather_moments(FakeFit())
    sh.reduce_minmax("mm")
    assert calls == [("allgather", "local", "all"), ("allreduce", "mm", "max")]
    with pytest.raises(RuntimeError, match="needs a Comm"):
        plain = _Sharded(None)
        plain.world = 2
        plain.capture()
