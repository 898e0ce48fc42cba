"""Function registry of the drop-in API (bg/registry.py:1-32).

Two kinds of ids live here, as in the reference:
  * operation ids ("distla.cholesky", "core.apply", ...) -> host functions
    that drive libbgp kernels on the device store (runtime.py / distla/ops.py);
  * generator ids ("gen.matern-nugget.cov", ...) -> `DeviceGenerator`
    descriptions of a built-in device kernel.

A Python callable registered as a generator is accepted by `register` (API
compatibility) but cannot run on the device: constructing with it raises
UnknownFunction.  There is no CPU fallback.
"""

from dataclasses import dataclass

from .errors import UnknownFunction

_FUNCTIONS = {}


@dataclass(frozen=True)
class DeviceGenerator:
    """A generator id bound to a device kernel (include/bgp.h BGP_GEN_*)."""

    family: int        # BGP_GEN_*
    part: int          # BGP_PART_*
    nugget: bool       # add theta[-1] where global i == j (cov part only)
    corr: str = ""     # "matern" | "sqexp" | "" (for reporting)


def register(fn_id, fn=None):
    """Register `fn` under `fn_id`; usable as a decorator."""
    if fn is None:
        def deco(f):
            _FUNCTIONS[fn_id] = f
            return f
        return deco
    _FUNCTIONS[fn_id] = fn
    return fn


def lookup(fn_id):
    try:
        return _FUNCTIONS[fn_id]
    except KeyError:
        raise UnknownFunction(f"no registered function {fn_id!r}") from None


def is_registered(fn_id):
    return fn_id in _FUNCTIONS


def device_generator(fn_id):
    """The device kernel behind a generator id, or UnknownFunction."""
    g = _FUNCTIONS.get(fn_id)
    if isinstance(g, DeviceGenerator):
        return g
    if g is None:
        raise UnknownFunction(f"no registered function {fn_id!r}")
    raise UnknownFunction(
        f"generator {fn_id!r} is a host callable; the b200 backend only runs "
        "built-in device generators (no CPU fallback)")
