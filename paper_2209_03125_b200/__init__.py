"""B200-native SAGE checksum hot path (arXiv 2209.03125)."""
