"""histgnn.cache conventions (cache.py:41-369) over the device cache.

The device `HistCache` already takes and returns numpy at `lookup` /
`update_cache` and exposes `.layers[l].row_of / admit_iter / row_owner /
capacity / _grow`; the one reference-visible attribute it keeps on the device
is the layer-0 feature region, which a reference caller reads as a numpy
array (`cache.feature_table`, cache.py:338-351).
"""

from __future__ import annotations

from ..cache import CachePolicy
from ..cache import HistCache as _DeviceHistCache
from ..graphs import _np

__all__ = ["CachePolicy", "HistCache"]


class HistCache(_DeviceHistCache):
    @property
    def feature_table(self):
        t = self.__dict__.get("_feature_table_dev")
        return None if t is None else _np(t)

    @feature_table.setter
    def feature_table(self, value):
        self.__dict__["_feature_table_dev"] = value

    @property
    def feature_table_dev(self):
        return self.__dict__.get("_feature_table_dev")
