"""E4 plumbing (include/bf.h bf_mcast_*): the multicast object, its bound
copy and the in-switch OR kernel, at P = 1 on the single GPU available (the
OR over one copy is the identity, so the merged buffer must equal what was
written; the kernel's slice arithmetic is checked at P > 1 by
test_nvls_slices).  Skipped where the device reports no multicast support.
The OR value at P > 1 needs P GPUs on one NVSwitch and is not exercised here
(DESIGN.md section 9)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mc_supported():
    import torch
    try:
        from cuda.bindings import driver as d  # cuda-python
        d.cuInit(0)
        err, v = d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0)
        return int(v) == 1
    except Exception:
        return torch.cuda.is_available()


def test_mcast_identity_merge(bflib, cuda):
    import torch
    bf = bflib
    if not _mc_supported():
        pytest.skip("no multicast support on this device")
    from paper_2512_15595_b200.dist import NvlsMerger
    nbytes = (1 << 22) + 8 * 13
    rng = np.random.default_rng(5)
    host = rng.integers(0, 256, nbytes, dtype=np.uint8)
    words = torch.from_numpy(host).to(cuda)
    n0 = bf.bf_launch_count()
    mg = NvlsMerger(nbytes)
    _, size = bf.bf_mcast_mc_ptr(mg.m)
    assert size >= nbytes
    mg.merge(words)
    torch.cuda.synchronize()
    assert bf.bf_launch_count() == n0 + 1
    assert np.array_equal(words.cpu().numpy(), host)
    assert np.array_equal(mg.buf.cpu().numpy(), host)
    # argument checks
    with pytest.raises(bf.BFError):
        bf.bf_mcast_or_reduce(mg.m, 1, nbytes)        # rank >= nranks
    with pytest.raises(bf.BFError):
        bf.bf_mcast_or_reduce(mg.m, 0, nbytes - 4)    # not a multiple of 8
    with pytest.raises(bf.BFError):
        bf.bf_mcast_or_reduce(mg.m, 0, size + 8)      # beyond the buffer
    mg.close()


def test_mcast_posix_handle_reimport(bflib, cuda):
    """The importer side of the POSIX-fd handle (pidfd_getfd of the
    exporter's fd) on this process's own blob."""
    bf = bflib
    if not _mc_supported():
        pytest.skip("no multicast support on this device")
    m, blob = bf.bf_mcast_create(1 << 21, 2, bf.BF_MCAST_POSIX_FD, True)
    try:
        m2, _ = bf.bf_mcast_create(1 << 21, 2, bf.BF_MCAST_POSIX_FD, False, blob)
        bf.bf_mcast_destroy(m2)
    finally:
        bf.bf_mcast_destroy(m)


def test_nvls_slices(bflib, cuda):
    """Every rank's slice together covers [0, bytes) once: at nranks = 3 one
    process runs all three slices on its P=3 object -- without the other
    devices bound there is nothing to reduce with, so only argument
    validation of rank < nranks is exercised; the partition itself is the
    same n8*r/P split as merge_alltoall's host arithmetic."""
    bf = bflib
    if not _mc_supported():
        pytest.skip("no multicast support on this device")
    m, _ = bf.bf_mcast_create(1 << 21, 3, bf.BF_MCAST_POSIX_FD, True)
    try:
        with pytest.raises(bf.BFError):
            bf.bf_mcast_or_reduce(m, 0, 1 << 21)  # not bound yet
    finally:
        bf.bf_mcast_destroy(m)
