"""K2 (tcgen05 kind::i8 association GEMM) must be EXACT: every operand is an
integer and the int32 tensor-core accumulation cannot round, so the result is
compared bit-for-bit with a float64 product of the same integers (all partial
sums are far below 2**53)."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

KWH = 32385


def _run(c_pad, p_pad, k_pad, seed=0):
    from paper_2604_21095_b200 import _native

    lib = _native.load_library()
    d = torch.device("cuda:0")
    g = torch.Generator(device=d).manual_seed(seed)
    qh = torch.randint(-127, 128, (p_pad, k_pad), generator=g, device=d, dtype=torch.int8)
    q1 = torch.randint(-127, 128, (p_pad, k_pad), generator=g, device=d, dtype=torch.int8)
    q0 = torch.randint(-63, 64, (p_pad, k_pad), generator=g, device=d, dtype=torch.int8)
    v = torch.randint(-1, 2, (c_pad, k_pad), generator=g, device=d, dtype=torch.int8)
    v127 = (v.to(torch.int16) * 127).to(torch.int8)
    x = torch.empty(c_pad, p_pad, dtype=torch.float64, device=d)
    st = torch.cuda.current_stream().cuda_stream
    _native.check(lib.pg_debug_assoc_gemm(
        qh.data_ptr(), q1.data_ptr(), q0.data_ptr(), p_pad, v.data_ptr(), v127.data_ptr(),
        c_pad, k_pad, x.data_ptr(), st))
    torch.cuda.synchronize()
    vd = v.double()
    q = KWH * qh.double() + 127 * q1.double() + q0.double()
    ref = vd @ q.T
    return x, ref


@pytest.mark.parametrize("c_pad,p_pad,k_pad", [(256, 256, 64), (512, 256, 1024), (768, 512, 23040)])
def test_gemm_exact(c_pad, p_pad, k_pad):
    x, ref = _run(c_pad, p_pad, k_pad)
    assert torch.equal(x, ref)
