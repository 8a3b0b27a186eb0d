"""NCCL paths on one GPU (world size 1 — this pool gives one GPU per call; the
N > 1 partitions are covered by the gloo tests in test_dist_gloo.py and the
rank/slab rule below): the C-ABI's NCCL-aware entries (st_fcs_dense_nccl,
st_fcs_cp_nccl) over a communicator the library creates, and the Python
restart-sharded RTPM under torch.distributed's NCCL backend (its exchange
buffer must live on the device: NCCL rejects host tensors)."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L
from paper_2106_13062_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(cuda):
    lib = L.lib()
    uid = (C.c_char * lib.st_nccl_unique_id_bytes())()
    L.check(lib.st_nccl_get_unique_id(uid))
    c = C.c_void_p()
    L.check(lib.st_nccl_comm_init_rank(C.byref(c), 1, uid, 0))
    yield c
    L.check(lib.st_nccl_comm_destroy(c))


def test_fcs_dense_nccl_world1(cuda, comm):
    lib = L.lib()
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 30, 20))
    dims = [64, 30, 20]
    fams = st.families_for(dims, st.EstimatorConfig(200, 3, 9))
    t = torch.from_numpy(x.ravel(order="F").copy()).cuda()
    packed = st.packed_families(fams)
    dims_a, lens_a = L.size_array(dims), L.size_array([200] * 3)
    lo, cnt = C.c_size_t(), C.c_size_t()
    L.check(lib.st_shard_range(20, 0, 1, C.byref(lo), C.byref(cnt)))
    assert (lo.value, cnt.value) == (0, 20)
    ws = lib.st_fcs_dense_workspace(L.ST_F64, 3, dims_a, cnt.value, 3, lens_a)
    wbuf = torch.empty(max(ws, 1), dtype=torch.uint8, device="cuda")
    out = torch.empty((3, fams[0].composed_len()), dtype=torch.float64, device="cuda")
    L.check(lib.st_fcs_dense_nccl(L.ST_F64, C.c_void_p(t.data_ptr()), 3, dims_a, 3,
                                  C.c_void_p(packed.data_ptr()), lens_a,
                                  C.c_void_p(out.data_ptr()), C.c_void_p(wbuf.data_ptr()), ws,
                                  comm, None))
    want = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams)
    torch.cuda.synchronize()
    assert torch.allclose(out, want, rtol=1e-12, atol=1e-12 * float(want.abs().max()))


def test_fcs_cp_nccl_world1(cuda, comm):
    lib = L.lib()
    rng = np.random.default_rng(4)
    dims, R = [40, 30, 20], 6
    fs = [rng.standard_normal((d, R)) for d in dims]
    w = rng.standard_normal(R)
    cp = st.CpTensor(w, fs)
    fams = st.families_for(dims, st.EstimatorConfig(300, 2, 5))
    packed = st.packed_families(fams)
    dims_a, lens_a = L.size_array(dims), L.size_array([300] * 3)
    ws = lib.st_fcs_cp_workspace(3, dims_a, R, 2, lens_a)
    wbuf = torch.empty(max(ws, 1), dtype=torch.uint8, device="cuda")
    out = torch.empty((2, fams[0].composed_len()), dtype=torch.float64, device="cuda")
    fptrs = (C.c_void_p * 3)(*[f.data_ptr() for f in cp._factors_cm])
    L.check(lib.st_fcs_cp_nccl(C.c_void_p(cp.weights.data_ptr()), R, 3, dims_a, fptrs, 2,
                               C.c_void_p(packed.data_ptr()), lens_a, C.c_void_p(out.data_ptr()),
                               C.c_void_p(wbuf.data_ptr()), ws, comm, None))
    want = st.fcs_cp_batched(cp, fams)
    torch.cuda.synchronize()
    assert torch.allclose(out, want, rtol=1e-12, atol=1e-12 * float(want.abs().max()))


def test_sharded_rtpm_nccl_backend(cuda):
    """dist.sharded_rtpm under the NCCL process group (advisor round 1: the
    all-gather buffer was a host tensor, which NCCL rejects)."""
    import torch.distributed as dist
    from paper_2106_13062_b200 import dist as pdist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29877")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        q = np.linalg.qr(np.random.default_rng(23).standard_normal((20, 2)))[0]
        t = configs.densify([3.0, 1.5], [q, q, q])
        est = st.EstimatorConfig(200, 3, 5)
        w, f = pdist.sharded_rtpm(st.FcsEngine(st.DenseTensor.from_array(t), est), 20, 2, 4, 6, 5)
        cp = st.rtpm(st.DenseTensor.from_array(t),
                     st.RtpmConfig(2, 4, 6, st.SketchBackend.FCS, est))
        np.testing.assert_allclose(w, cp.weights.cpu().numpy(), rtol=1e-9)
        np.testing.assert_allclose(f, cp.factors[0].cpu().numpy(), rtol=1e-9, atol=1e-12)
    finally:
        dist.destroy_process_group()
