"""The drop-in shim rebinds the reference's hot-path names in the defining
AND the caller modules.  Needs the reference tree (present in
the build container only); no compute is run."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not mounted")
def test_install_patches_callers_and_uninstall_restores():
    sys.path.insert(0, REF)
    try:
        import lsrm
        import lsrm.recon_pipeline as rp
        import lsrm.seq_parallel as sp
        from paper_2604_05182_b200 import dropin
        import paper_2604_05182_b200 as ours
        ref_nsa = rp.nsa_cross_attention
        ref_sel = sp.sel_attention
        patched = dropin.install(lsrm)
        try:
            names = {(m, n) for m, n in patched}
            assert ("lsrm.nsa_attention", "nsa_cross_attention") in names
            assert ("lsrm.recon_pipeline", "nsa_cross_attention") in names   # caller module
            assert ("lsrm.seq_parallel", "sel_attention") in names
            assert ("lsrm.seq_parallel", "shard_blocks") in names
            assert ("lsrm.runner", "build_routing_plan") in names
            assert rp.nsa_cross_attention is ours.nsa_cross_attention
            assert sp.sel_attention is ours.sel_attention
        finally:
            dropin.uninstall()
        assert rp.nsa_cross_attention is ref_nsa and sp.sel_attention is ref_sel
    finally:
        sys.path.remove(REF)
