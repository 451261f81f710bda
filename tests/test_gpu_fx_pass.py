"""The automatic Echo pass on arbitrary PyTorch models on
the GPU: the EchoModule's loss and every parameter gradient are bitwise those of the unmodified model
(Echo changes no math), the bytes its saved-tensor hooks actually keep equal the
estimator's Echo plan exactly, and the unmodified model's autograd keeps exactly the estimator's
Baseline bytes (reading R11's per-op rules are torch's)."""
import pytest
import torch

from tests.fx_models import GatedNet, ResMLP, ReluTaps, ResConvNet
from tests.gpu_util import bits_equal

pytestmark = pytest.mark.gpu


def _grads(m):
    return [p.grad.detach().clone() for p in m.parameters()]


@pytest.mark.parametrize("make,shape", [(lambda: GatedNet(64, 3, 0.2), (32, 64)), (lambda: ResMLP(128, 4), (16, 128)),
                                        (lambda: ReluTaps(256, 5), (64, 256)), (lambda: GatedNet(512, 2, 0.1), (256, 512)),
                                        (lambda: ResConvNet(16, 2), (4, 3, 32, 32))],
                         ids=["gated", "resmlp", "relutaps", "gated-wide", "resconv"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
def test_echo_module_bitwise_and_bytes(make, shape, dtype, cuda_dev):
    from paper_1805_08899_b200 import fx_pass as X
    torch.backends.cudnn.deterministic = True                    # deterministic conv gradients for the bitwise check
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(0)
    m = make().to("cuda", dtype)
    x = torch.randn(*shape, device="cuda", dtype=dtype)
    torch.manual_seed(123)
    ref, base_bytes = X.baseline_saved_bytes(m, x)                # unmodified model (dropout draws from seed 123)
    ref.backward()
    g_ref = _grads(m)
    m.zero_grad(set_to_none=True)
    em = X.EchoModule(m, (x,))
    base = X.EchoPlan(m, (x,), strategy="baseline")
    assert base_bytes == base.stash_bytes(), (base_bytes, base.stash_bytes())
    torch.manual_seed(123)                                        # the same dropout draws
    loss = em(x)
    kept = em.kept_bytes()
    assert kept == em.plan.stash_bytes(), (kept, em.plan.stash_bytes())
    assert kept <= base_bytes
    loss.backward()
    assert bits_equal(loss.detach(), ref.detach())
    for a, b in zip(_grads(m), g_ref):
        assert bits_equal(a, b)
    # a second step reuses the plan (fresh bookkeeping per forward)
    m.zero_grad(set_to_none=True)
    torch.manual_seed(123)
    em(x).backward()
    for a, b in zip(_grads(m), g_ref):
        assert bits_equal(a, b)


def test_sign_pack_roundtrip(cuda_dev):
    from paper_1805_08899_b200 import abi
    abi.load()
    for dt in (torch.float32, torch.bfloat16, torch.bool, torch.uint8):
        n = 1003
        x = torch.randn(n, device="cuda")
        x = (x > 0.3) if dt == torch.bool else (x > 0.3).to(torch.uint8) if dt == torch.uint8 else x.to(dt)
        bits = torch.empty((n + 7) // 8, dtype=torch.uint8, device="cuda")
        abi.echo_sign_pack(x, bits)
        out = torch.empty(n, dtype=dt, device="cuda")
        abi.echo_bits_unpack(bits, out)
        ref = (x > 0) if dt not in (torch.bool, torch.uint8) else (x != 0)
        assert torch.equal(out.bool() if dt != torch.bool else out, ref)
