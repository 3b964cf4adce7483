"""The one-to-many fan-out step (csrc/fanout.cu) on this pool's one-GPU
slice: the capability report says why NVSwitch multicast is not available
(one device, no fabric manager) and the broadcast falls back to peer copies;
every destination receives the source bytes exactly.  With real devices the
same call takes the multicast path (multimem.st through one multicast object
binding every destination's pages)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200 import _lib
from paper_2404_14691_b200 import device as D

pytestmark = pytest.mark.gpu


def land_pattern(gpu, nbytes, seed):
    data = O.db_bytes(seed, nbytes)
    seg = D.pool_alloc(gpu, nbytes, _lib.CLASS_READ_ONLY)
    op = D.load(gpu, seg.dptr, data, None)
    op.wait()
    op.release()
    return seg, data


@pytest.mark.parametrize("planes", [1, 3])
def test_broadcast_reaches_every_plane(built, planes):
    from conftest import gpu_available
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    flags = _lib.SAGE_INIT_PEER_ACCESS | (_lib.SAGE_INIT_SHARE_DEVICE if planes > _lib.device_count() else 0)
    _lib.init(n_gpus=planes, pool_bytes=8 << 30, staging_bytes=32 << 20, chunk_bytes=4 << 20, flags=flags)
    try:
        caps = D.fanout_caps()
        assert caps["n_gpus"] == planes and caps["why"]
        full = (1 << planes) - 1
        assert all(m == full for m in caps["peer_mask"])          # every plane reaches every other's pages
        if caps["n_devices"] < planes or caps["n_devices"] < 2:
            assert not caps["multicast"]                          # multicast needs one plane per device
        nbytes = 3 << 20
        src, data = land_pattern(0, nbytes, 11)
        dsts = [(g, D.pool_alloc(g, nbytes, _lib.CLASS_READ_ONLY)) for g in range(planes)]
        path, ev = D.fanout_broadcast(0, src.dptr, nbytes, dsts)
        ev.sync()
        ev.release()
        assert path in ("multicast", "p2p")
        if not caps["multicast"]:
            assert path == "p2p"
        for g, seg in dsts:
            assert np.array_equal(D.read_device(g, seg.dptr, nbytes), data), (g, path)
        # forced peer copies give the same bytes
        path2, ev = D.fanout_broadcast(0, src.dptr, nbytes, dsts[-1:], p2p_only=True)
        ev.sync()
        ev.release()
        assert path2 == "p2p"
        with pytest.raises(_lib.SageError):                       # bytes must be a multiple of 16
            D.fanout_broadcast(0, src.dptr, nbytes - 1, dsts)
        for _, seg in dsts:
            seg.free()
        src.free()
    finally:
        _lib.shutdown()
