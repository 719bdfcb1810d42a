import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ctx():
    import paper_2502_08246_b200 as sb
    return sb.default_context()


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(autouse=True)
def _step_state_clean(request):
    """After every GPU test the default context's per-step counters and flags
    must be re-armed (zero): a leak would corrupt the next decode step."""
    yield
    if request.node.get_closest_marker("gpu") is None or not _has_gpu():
        return
    import paper_2502_08246_b200 as sb
    if sb._default_ctx is None:
        return
    st = sb._default_ctx.step_state()
    assert not any(st.values()), f"step state leaked: {st}"
