"""B200-native AMG-PCG hot path for H(curl) (arXiv 2602.23613)."""
