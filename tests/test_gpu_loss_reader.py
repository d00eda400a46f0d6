"""model.LossReader: pipelined per-step loss reads (bench.py's e2e loop) return every pushed value in
order, even when the device tensor is overwritten by the next step before the host reads."""
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import model


def test_loss_reader_pipelined_values():
    loss = torch.zeros((), device="cuda")
    r = model.LossReader(2)
    got = []
    for i in range(5):
        torch.cuda._sleep(2_000_000)  # the "step" is still running when the host moves on
        loss.fill_(float(i) + 0.5)
        r.push(loss)
        if i:
            got.append(r.pop())
    got.append(r.pop())
    assert got == [i + 0.5 for i in range(5)]
    r.push(loss)
    r.push(loss)
    with pytest.raises(RuntimeError):
        r.push(loss)
