"""pytest plugin: run the REFERENCE's own test-suite against this framework.

Loaded with `-p fmmb_ref_bridge` before collection: binds the B200 kernel
plugin as `fmmkit.backend.kernels` (the reference's own swap mechanism,
cli.py:263-266) and replaces the build API entry points the tests import
(`from fmmkit import build_all, sort_points, ...`), the scan, the FMMS
container IO and dump/load_structures with the device versions.
Test infrastructure only.
"""

import fmmkit
import fmmkit.backend as _backend
import fmmkit.lists as _lists
import fmmkit.pseudosort as _pseudosort

import paper_1301_1704_b200 as fb
from paper_1301_1704_b200 import kernels as _kernels

_backend.kernels = _kernels
for _name in ("build_all", "sort_points", "histogram_and_sort_index", "reorder",
              "build_bookmarks", "build_neighbor_table", "build_level_directory",
              "build_translation_stencils", "propagate_to_parents", "choose_max_level"):
    _obj = getattr(fb, _name)
    setattr(fmmkit, _name, _obj)
    for _mod in (_lists, _pseudosort):
        if hasattr(_mod, _name):
            setattr(_mod, _name, _obj)

import fmmkit.scan as _scan  # noqa: E402

for _name in ("exclusive_scan", "compact_flags"):  # scan.py:25-81 -> device scan
    setattr(fmmkit, _name, getattr(fb, _name))
    setattr(_scan, _name, getattr(fb, _name))

import fmmkit.container as _container  # noqa: E402

from paper_1301_1704_b200 import container as _our_container  # noqa: E402

for _name in ("Section", "write_container", "read_container"):  # container.py -> streaming IO
    setattr(_container, _name, getattr(_our_container, _name))
for _name in ("dump_structures", "load_structures"):  # lists.py:203-257
    setattr(fmmkit, _name, getattr(fb, _name))
    setattr(_lists, _name, getattr(fb, _name))
import fmmkit.boxtype as _boxtype  # noqa: E402

from paper_1301_1704_b200 import boxtype as _our_boxtype  # noqa: E402

for _name in ("classify", "dump_typed", "load_typed"):  # boxtype.py -> device classify
    setattr(_boxtype, _name, getattr(_our_boxtype, _name))
fmmkit.classify = _our_boxtype.classify

import fmmkit.partition as _partition  # noqa: E402

from paper_1301_1704_b200 import partition as _our_partition  # noqa: E402

for _name in ("choose_partition", "dump_plan", "load_plan"):  # partition.py:74-257
    setattr(_partition, _name, getattr(_our_partition, _name))
fmmkit.choose_partition = _our_partition.choose_partition
# near_field_potentials / direct_sum (fmm.py) reach the device through the
# bound plugin: kernels.near_field / kernels.direct_potentials

CALLS = {"build_all": 0}
_orig_build_all = fb.build_all


def _counting_build_all(*a, **k):
    CALLS["build_all"] += 1
    return _orig_build_all(*a, **k)


fmmkit.build_all = _counting_build_all
_lists.build_all = _counting_build_all


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"fmmb_ref_bridge: build_all calls routed to the B200 build: "
                                f"{CALLS['build_all']}")
