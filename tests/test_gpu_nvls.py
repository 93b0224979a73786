"""E4 plumbing (include/bf.h bf_mcast_*): the multicast object, its bound
copy and the in-switch OR kernel, at P = 1 on the single GPU available (the
OR over one copy is the identity, so the merged buffer must equal what was
written; the kernel's slice arithmetic is checked at P > 1 by
test_nvls_slices).  Skipped where the device reports no multicast support.
The OR value at P > 1 needs P GPUs on one NVSwitch and is not exercised here
(DESIGN.md section 9).  test_mcast_unavailable_is_reported runs
everywhere: where the driver refuses multicast objects the C ABI must say
so with an error code, never crash or silently succeed."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mc_supported(bf):
    """Multicast objects can be created here.  The device attribute alone is
    not enough: in a container that exposes one GPU of an NVSwitch node the
    driver reports MULTICAST_SUPPORTED = 1 yet refuses cuMulticastCreate
    (CUDA_ERROR_INVALID_VALUE for every numDevices and handle type,
    tools/check_mc2.py)."""
    try:
        m, _ = bf.bf_mcast_create(1 << 21, 1, bf.BF_MCAST_POSIX_FD, True)
    except bf.BFError:
        return False
    bf.bf_mcast_destroy(m)
    return True


def test_mcast_identity_merge(bflib, cuda):
    import torch
    bf = bflib
    if not _mc_supported(bf):
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
    if not _mc_supported(bf):
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
    if not _mc_supported(bf):
        pytest.skip("no multicast support on this device")
    m, _ = bf.bf_mcast_create(1 << 21, 3, bf.BF_MCAST_POSIX_FD, True)
    try:
        with pytest.raises(bf.BFError):
            bf.bf_mcast_or_reduce(m, 0, 1 << 21)  # not bound yet
    finally:
        bf.bf_mcast_destroy(m)


def test_mcast_unavailable_is_reported(bflib, cuda):
    bf = bflib
    for args in [(0, 1, bf.BF_MCAST_POSIX_FD), (1 << 21, 0, bf.BF_MCAST_POSIX_FD), (1 << 21, 1, 7)]:
        with pytest.raises(bf.BFError) as ei:
            bf.bf_mcast_create(*args, True)
        assert ei.value.code == bf.BF_EINVAL
    try:
        m, blob = bf.bf_mcast_create(1 << 21, 1, bf.BF_MCAST_POSIX_FD, True)
    except bf.BFError as e:
        assert e.code in (bf.BF_ECUDA, bf.BF_EUNSUPPORTED)
        assert "cuMulticastCreate" in str(e) or "multicast" in str(e)
        return
    assert len(blob) == bf.BF_MCAST_HANDLE_BYTES
    bf.bf_mcast_destroy(m)
