"""Route an installed reference package (``fuzzdepth``) to the B200 kernels.

This is the module-swap a maintainer would add to the reference
(INTEGRATION.md §2): every depth-path function of ``fuzzdepth`` -- the public
ones (depth.py:192-363, inclusion.py:22-107) and the internal seams
(reduction.py:36-97 ``weighted_sum``/``weighted_inner``/``weighted_excess``/
``gram_block``, depth.py:88-102 ``member_masses``, depth.py:231-243
``_member_mean_terms``) -- is rebound to this package's implementation in
every ``fuzzdepth`` module that imported it by name (the CLI, consistency
and bench modules bind ``depth_by_method`` at import time), so the
reference's own callers and tests run on the GPU unchanged.

    import fuzzdepth, paper_2512_15187_b200.integration as I
    I.install(fuzzdepth)          # ... I.uninstall() restores the originals
"""
from __future__ import annotations

import sys

# (reference module, name) -> replacement attribute of this package
_ROUTES = {
    "depth": ("depth_pid", "depth_pid_mean", "depth_eid", "depth_by_method",
              "depth_similarity_baseline", "compare_pid_vs_mean", "member_masses",
              "_member_mean_terms"),
    "inclusion": ("prob_inclusion", "subset_epsilon", "fuzzy_dice", "prob_iou"),
    "reduction": ("gram_block", "weighted_sum", "weighted_inner", "weighted_excess"),
}

_saved: dict = {}


def _replacement(name: str):
    from . import depth, inclusion, reduction

    for mod in (depth, inclusion, reduction):
        if hasattr(mod, name):
            return getattr(mod, name)
    raise AttributeError(name)


def install(fd=None) -> list[str]:
    """Rebind the depth path of ``fd`` (default: ``import fuzzdepth``) to the
    B200 implementation; returns the rebound ``module.name`` list."""
    if fd is None:
        import fuzzdepth as fd  # noqa: F811
    if _saved:  # already installed: keep the true originals for uninstall()
        return sorted(f"{m}.{n}" for m, n in _saved)
    base = fd.__name__
    originals = {}
    for sub, names in _ROUTES.items():
        mod = sys.modules.get(f"{base}.{sub}")
        if mod is None:
            continue
        for nm in names:
            if hasattr(mod, nm):
                originals[nm] = getattr(mod, nm)
    done = []
    for modname, mod in list(sys.modules.items()):
        if mod is None or not (modname == base or modname.startswith(base + ".")):
            continue
        for nm, orig in originals.items():
            if getattr(mod, nm, None) is orig:
                _saved[(modname, nm)] = orig
                setattr(mod, nm, _replacement(nm))
                done.append(f"{modname}.{nm}")
    return sorted(done)


def uninstall() -> None:
    """Restore every attribute ``install`` rebound."""
    for (modname, nm), orig in list(_saved.items()):
        mod = sys.modules.get(modname)
        if mod is not None:
            setattr(mod, nm, orig)
    _saved.clear()
