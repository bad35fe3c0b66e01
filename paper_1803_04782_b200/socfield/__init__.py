"""`socfield` — Python surface of the B200 (CUDA, sm_100a) build of the discrete social-field
pedestrian engine.  Drop-in for the reference package of the same name: same functions, classes
and exceptions (reference proj/python/socfield/__init__.py, proj/bindings/module.cpp).

Import with ``paper_1803_04782_b200`` on ``sys.path`` ahead of any other ``socfield``::

    import paper_1803_04782_b200.socfield as socfield      # or
    from paper_1803_04782_b200 import socfield
"""
from ._core import *  # noqa: F401,F403
from ._core import __doc__, _kind_table, backend, device_count  # noqa: F401
