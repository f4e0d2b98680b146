"""pytest plugin: run the reference's own unit tests against this backend (compat mode).

    PYTHONPATH=<repo>:<repo>/tests:baseline/_ref python -m pytest -p compat_plugin <reference tests>/test_tensor.py

Installs paper_2409_11600_b200.nsk_backend.install_compat() before the reference test modules are collected,
so their ``from nsk.tensor import ...`` / ``from nsk import autodiff`` bindings resolve to the device backend.
"""


def pytest_configure(config):
    from paper_2409_11600_b200.nsk_backend import install_compat

    install_compat()
