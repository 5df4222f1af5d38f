"""B200-native recursive skeletonization (arXiv 2001.11619)."""
