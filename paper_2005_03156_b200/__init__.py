"""B200-native point-to-block projection (arXiv 2005.03156, "Fast Mapping
onto Census Blocks"): a GPU cell index over leaf polygons and an exact fp64
crossing-number lookup, behind the reference's build_cover / query_leaves
interface.  See DESIGN.md."""
from .fastmap import (AssignmentResult, CellIndex, CoverMode, CoverParams, LeafRegion,
                      PolygonGeometry, Soup, build_cover, build_index, build_trie,
                      exhaustive_assign, index_stats, leaves_to_soup, query, query_leaves,
                      validate_cover_params)

__all__ = [
    "AssignmentResult", "CellIndex", "CoverMode", "CoverParams", "LeafRegion",
    "PolygonGeometry", "Soup", "build_cover", "build_index", "build_trie",
    "exhaustive_assign", "index_stats", "leaves_to_soup", "query", "query_leaves",
    "validate_cover_params",
]
