"""B200-native Wolstenholme / Vandiver residue search (arXiv:2101.11157 hot path)."""
