"""The reference-side binding: route a running
``mvdtw`` (the reference package) through the B200 search.

``mvdtw.cli`` binds ``nn_search`` by name at import (cli.py:34) and
``mvdtw.search._run_sample`` resolves the module global (search.py:193), so a
drop-in replaces both.  ``patch_mvdtw`` does that with a wrapper that
translates the reference's ``SearchParams`` / ``Method`` into this package's
(same fields, defaults and values) and returns the reference's own
``NnOutcome`` type, so tuning, selection and the CLI keep working unchanged.
"""

from __future__ import annotations

_PARAM_FIELDS = ("window", "refresh_period", "trigger_ti", "trigger_pc", "quant_levels", "max_boxes",
                 "group_width", "min_cell_frac", "dims_used")


def translate_params(ref_params):
    """mvdtw.SearchParams -> paper_2101_07731_b200.SearchParams (core.py:154-198)."""
    from .core import SearchParams

    kw = {f: getattr(ref_params, f) for f in _PARAM_FIELDS if hasattr(ref_params, f)}
    return SearchParams(method=getattr(ref_params.method, "value", ref_params.method), **kw)


def translate_method(ref_method):
    """mvdtw.Method (or None) -> this package's Method (or None)."""
    from .core import Method

    return None if ref_method is None else Method(getattr(ref_method, "value", ref_method))


def make_nn_search(outcome_type, impl=None):
    """An ``nn_search(query, candidates, params, advanced=None,
    dim_range=None)`` with the reference's signature, computed by ``impl``
    (default: this package's GPU ``nn_search``) and returning ``outcome_type``
    (the reference's NnOutcome)."""
    from . import search

    impl = impl or search.nn_search

    def nn_search(query, candidates, params, advanced=None, dim_range=None):
        out = impl(query, candidates, translate_params(params), advanced=translate_method(advanced),
                   dim_range=dim_range)
        return outcome_type(**vars(out))

    return nn_search


def patch_mvdtw(search_module, cli_module=None, impl=None):
    """Install the GPU nn_search into ``mvdtw.search`` (and ``mvdtw.cli``
    when given); returns the installed function."""
    fn = make_nn_search(search_module.NnOutcome, impl)
    search_module.nn_search = fn
    if cli_module is not None:
        cli_module.nn_search = fn
    return fn
