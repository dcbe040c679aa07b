"""B200-native YAND-MVSK sample-oracle core (arXiv 2604.25378 hot path)."""
