"""Conformance shim: run the reference package ``bigwht`` with every
butterfly on the B200.

The reference modules import ``fwht_array`` and ``check_magnitude_bound``
by name (core.py:97,80; parallel.py:20; external.py:31; noisy.py:19), so
``install()`` rebinds those module attributes to this package's drop-ins:

* ``bigwht.fwht_inplace`` / ``inverse_wht_inplace`` (core.py:120-173),
  ``run_parallel``'s chunk phase (parallel.py:151), the external initial
  pass (external.py:253) and the noise check (noisy.py:254) then call the
  GPU transform; numpy buffers are staged through HBM in the same call;
* the bound check (core.py:80-94, parallel.py:175, noisy.py:113) runs as a
  device reduction;
* this package's exceptions become subclasses of their ``bigwht.errors``
  namesakes (errors.bind_reference), so the reference's
  ``pytest.raises(OverflowBoundError)`` and cli.py:577-579's
  ``except BigWHTError`` (exit code 3) catch what the GPU path raises.

The reference's own control flow (domains, phase barriers, disk I/O) is
untouched.  As a pytest plugin (``pytest -p paper_1607_01039_b200.shim``)
the shim is installed before the reference's test modules are imported,
so their ``from bigwht.core import fwht_array`` binds the GPU function.
"""

from __future__ import annotations

import importlib

from . import core, errors

_PATCHED_MODULES = ("bigwht", "bigwht.core", "bigwht.parallel", "bigwht.external", "bigwht.noisy")
_ATTRS = {"fwht_array": core.fwht_array, "check_magnitude_bound": core.check_magnitude_bound}

installed = False
calls = {"fwht_array": 0, "check_magnitude_bound": 0}  # how often the reference called into the B200 path


def _counting(name, fn):
    def wrapper(*args, **kwargs):
        calls[name] += 1
        return fn(*args, **kwargs)

    wrapper.__name__ = fn.__name__
    wrapper.__doc__ = fn.__doc__
    wrapper.__wrapped__ = fn
    return wrapper


def install() -> None:
    """Bind the reference's callers to the B200 path (idempotent).  Raises
    ImportError when ``bigwht`` is not importable."""
    global installed
    if installed:
        return
    ref_errors = importlib.import_module("bigwht.errors")
    if not errors.bind_reference(ref_errors):
        raise ImportError("bigwht.errors could not be bound")
    wrapped = {name: _counting(name, fn) for name, fn in _ATTRS.items()}
    for modname in _PATCHED_MODULES:
        mod = importlib.import_module(modname)
        for name, fn in wrapped.items():
            if hasattr(mod, name):
                setattr(mod, name, fn)
    installed = True


def pytest_configure(config) -> None:  # pytest plugin hook
    install()


def pytest_terminal_summary(terminalreporter) -> None:  # pytest plugin hook
    terminalreporter.write_line(
        "bigwht_b200 shim: fwht_array calls on the B200 = %d, check_magnitude_bound calls = %d"
        % (calls["fwht_array"], calls["check_magnitude_bound"]))
