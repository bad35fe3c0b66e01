"""Test configuration.

`-m "not gpu"`  — CPU suite: the C oracle against the golden vectors and against the compiled
                  reference (oracle/_ref), host logic of the product (tables, scenario parsing),
                  and the C-ABI export check.  Runs anywhere.
`-m gpu`        — parity tests proper: the CUDA engine (through the C ABI / host mirror) against
                  the oracle on identical inputs.  Needs a B200; never reads /root/reference.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _device_count() -> int:
    try:
        from paper_1803_04782_b200 import socfield

        return socfield.device_count()
    except Exception:
        return 0


def pytest_collection_modifyitems(config, items):
    if _device_count() > 0:
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import shim

    if not shim.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference; `make -C oracle ref`)")
    return shim.load_ref()


@pytest.fixture(scope="session")
def product_lib():
    from oracle import shim

    if not shim.have_product():
        pytest.fail("oracle/build/libsocfield_b200_shim.so missing: run "
                    "`python -m paper_1803_04782_b200.build` — the product has no CPU fallback")
    return shim.load_product()
