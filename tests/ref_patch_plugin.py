"""pytest plugin (-p ref_patch_plugin): before the reference's own test
modules are collected, import the reference package and rebind its hot path
onto libboba_b200 (paper_2306_10410_b200.integration.patch_reference)."""

import os
import sys


def pytest_configure(config):
    root = os.environ["BOBA_REPO_ROOT"]
    sys.path.insert(0, root)
    sys.path.insert(0, os.environ["BOBA_REF_SRC"])
    import boba  # the reference package

    from paper_2306_10410_b200.integration import patch_reference

    patch_reference(boba)
    config._boba_patched = True
