"""Install the GPU force calculator into the reference package (mdtune).

The reference resolves its force backend through module globals:
``mdtune.simulation.ForceCalculator`` (simulation.py:21,144),
``mdtune.dataset.ForceCalculator`` (dataset.py:21,114) and
``mdtune.containers.ForceCalculator`` (used by ``compute_forces``,
containers.py:494-511).  Its own tests swap the backend the same way
(tests/test_simulation.py:142-148, tests/test_dataset.py:101-110).

    import mdtune
    from paper_2505_03438_b200 import plugin
    plugin.install()          # every simulate()/gen-data/compute_forces now runs on the GPU
    ...
    plugin.uninstall()

As a pytest plugin (``pytest -p paper_2505_03438_b200.plugin``) the swap
happens in ``pytest_configure``, i.e. before test modules bind the name at
import time (tests/test_containers.py:9), so the reference's own test files
run against the GPU backend unchanged.
"""

from __future__ import annotations

import importlib

from .calculator import HostForceCalculator

_TARGETS = ("mdtune.simulation", "mdtune.dataset", "mdtune.containers")
_saved: dict = {}


def install(calculator_cls=HostForceCalculator) -> list:
    """Swap ForceCalculator in every reference module that binds it."""
    done = []
    for name in _TARGETS:
        try:
            mod = importlib.import_module(name)
        except ImportError:
            continue
        if hasattr(mod, "ForceCalculator"):
            _saved.setdefault(name, mod.ForceCalculator)
            mod.ForceCalculator = calculator_cls
            done.append(name)
    return done


def uninstall() -> None:
    for name, cls in _saved.items():
        mod = importlib.import_module(name)
        mod.ForceCalculator = cls
    _saved.clear()


def pytest_configure(config):   # pragma: no cover - exercised under pytest -p
    config._mdg_installed = install()


def pytest_report_header(config):   # pragma: no cover - exercised under pytest -p
    """The swap, stated in the run's header so a log shows which backend ran."""
    import torch
    done = getattr(config, "_mdg_installed", [])
    dev = torch.cuda.get_device_name(0) if torch.cuda.is_available() else "no CUDA device"
    return [f"mdg plugin: ForceCalculator -> {HostForceCalculator.__module__}."
            f"{HostForceCalculator.__name__} in {', '.join(done) or 'nothing'} ({dev})"]
