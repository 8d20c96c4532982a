"""Re-point the reference package's hot path at the B200 implementation.

    import undertext                                   # the reference package
    from paper_1612_06457_b200 import integrate
    integrate.install(undertext)                       # opt-in, reversible
    ...
    integrate.uninstall(undertext)

``install`` replaces, in every loaded ``undertext.*`` module, each name bound to
one of the reference's hot-path functions by the drop-in of the same name --
the modules that own them (``projection``, ``eigen``, ``annotations``,
``rendering``, ``stack``) and every module that imported them by name
(``pipeline`` binds ``fit``/``project_stack``/``rescale``/``compose_rgb``/
``assemble_matrix``/``normalize_stack`` at import time, ``estimators`` binds
``fit_cva``/``fit_lda``/``fit_pca``, ``cli`` binds ``project_stack`` ...).  The
reference's own ``fit`` dispatch and ``rescale`` stay and reach the drop-ins
through their module globals.  Inputs are duck-typed, so the reference's
DesignMatrix / SpectralStack / TrainingSet / ScorePlane / ProjectionModel
objects pass through unchanged; outputs are this package's mirror types, which
carry the same fields (and the same model JSON).

What is replaced (reference file:line -> drop-in):

* annotations.assemble_matrix (annotations.py:195)  -> K1 gather
* projection.compute_scatter (:172), standardize (:152), fit_cva (:211),
  fit_lda (:240), fit_pca (:273), fit_pca_unsupervised (:298),
  project_stack (:391)                               -> K1 / K2 / K3 / K4
* eigen.solve_gen_eig_sym (eigen.py:75)              -> K3
* rendering.rescale_full (:124), rescale_training_range (:133),
  rescale_percentile (:155), compose_rgb (:206)     -> K5 / select / compose
* stack.normalize_stack (stack.py:180)               -> normalize kernels
* pipeline.render_planes (pipeline.py:136)           -> one K4 pass + device codecs
* with ``codecs=True`` also rendering.save_image / load_image and
  stack.load_stack (device PNG / TIFF encode, TIFF decode).

There is no CPU fallback: on a machine without a CUDA device every replaced
function raises ``RuntimeError`` (tests/test_integration_cpu.py drives the
reference's own pipeline to exactly that point).
"""

from __future__ import annotations

import sys
import types

HOT_PATH = {
    "annotations": ("assemble_matrix",),
    "projection": ("compute_scatter", "standardize", "fit_cva", "fit_lda", "fit_pca",
                   "fit_pca_unsupervised", "project_stack"),
    "eigen": ("solve_gen_eig_sym",),
    "rendering": ("rescale_full", "rescale_training_range", "rescale_percentile",
                  "compose_rgb"),
    "stack": ("normalize_stack",),
    "pipeline": ("render_planes",),
}
CODECS = {
    "rendering": ("save_image", "load_image"),
    "stack": ("load_stack",),
}

_saved: dict[str, list] = {}


def _dropin(name: str):
    import paper_1612_06457_b200 as b

    if name == "standardize":
        from .projection import standardize
        return standardize
    return getattr(b, name)


def _package(undertext) -> str:
    if isinstance(undertext, types.ModuleType):
        return undertext.__name__
    return str(undertext or "undertext")


def install(undertext=None, codecs: bool = False) -> dict:
    """Re-point the reference's hot path (see the module docstring).
    Returns {qualified name: count of rebindings}.  Idempotent."""
    pkg = _package(undertext)
    __import__(pkg)
    for sub in set(HOT_PATH) | set(CODECS):
        __import__(f"{pkg}.{sub}")
    table = {k: list(v) for k, v in HOT_PATH.items()}
    if codecs:
        for k, v in CODECS.items():
            table.setdefault(k, []).extend(v)
    if pkg in _saved:
        uninstall(pkg)
    mods = [m for n, m in list(sys.modules.items())
            if m is not None and (n == pkg or n.startswith(pkg + "."))]
    saved, counts = [], {}
    for owner, names in table.items():
        owner_mod = sys.modules[f"{pkg}.{owner}"]
        for name in names:
            original = getattr(owner_mod, name)
            new = _dropin(name)
            n = 0
            for m in mods:
                if getattr(m, name, None) is original:
                    saved.append((m, name, original))
                    setattr(m, name, new)
                    n += 1
            counts[f"{owner}.{name}"] = n
    _saved[pkg] = saved
    return counts


def uninstall(undertext=None) -> None:
    """Restore every binding ``install`` changed."""
    pkg = _package(undertext)
    for m, name, original in reversed(_saved.pop(pkg, [])):
        setattr(m, name, original)
