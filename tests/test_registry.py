"""Spec / label layer, pinned like the reference (test_backends.py:33-41)."""

import ctypes

import pytest

from paper_2002_05599_b200 import registry
from paper_2002_05599_b200._lib import NsgSpec, make_spec
from paper_2002_05599_b200.errors import ConfigurationError
from paper_2002_05599_b200.registry import SorterSpec


def test_spec_field_order_is_pinned():
    assert SorterSpec._fields == (
        "kind", "family", "swap", "ins_variant", "base_kind", "rss_oversampling", "rss_block",
        "rss_threshold", "rss_sample_seed", "qs_base_is_rss", "qs_threshold", "qs_depth_factor",
        "qs_final_pass", "pivot_swap")
    assert [f for f, _ in NsgSpec._fields_][:14] == list(SorterSpec._fields)
    assert ctypes.sizeof(NsgSpec) == 18 * 4


@pytest.mark.parametrize("label", ["SN Best 4CmS", "SN BN-L ISwp", "SN BN-R TCOp", "IS Def",
                                   "RSS 332 SN Best 4CmS", "RSS 315 IS Def", "QS SN Best 4CmS", "StdSort"])
def test_label_round_trip(label):
    assert registry.format_label(registry.parse_label(label)) == label


def test_rss_defaults():
    sp = registry.spec_rss("332")
    assert (sp.rss_oversampling, sp.rss_block, sp.rss_threshold, sp.rss_sample_seed) == (3, 2, 16, 0x5EED)
    c = make_spec(sp)
    assert c.kind == 2 and c.rss_sample_seed == 0x5EED and c.key_dtype == registry.KEY_U64


@pytest.mark.parametrize("bad", ["", "SN Foo 4CmS", "SN Best XYZ", "RSS 732 SN Best 4CmS",
                                 "RSS 306 SN Best 4CmS", "RSS 302 IS Def", "IS Nope"])
def test_bad_labels(bad):
    with pytest.raises(ConfigurationError):
        registry.parse_label(bad)


def test_network_threshold_cap():
    with pytest.raises(ConfigurationError):
        registry.spec_rss("332", "SN Best 4CmS", threshold=17)
    registry.spec_rss("332", "IS Def", threshold=40)
