"""B200-native batched small-set sorter (arXiv 2002.05599's hot path on sm_100a).

Public surface mirrors the reference package `netsort`:
  smallsort.sort_network / sort_small / insertion_sort
  rss.RssConfig / rss_sort / select_splitters / classify_block
  backend.run_sorter_many / run_sorter / swap_pairs / classify_block_u64
plus the typed batch front ends batch.sort_rows / batch.sort_segments.
All sorting runs in libnsg.so (hand-written CUDA for sm_100a); importing the
package does not touch the GPU, calling a sorter without one raises.
"""

from . import errors, items, networks, registry, swaps  # noqa: F401

__version__ = "0.1.0"
