"""rnmf-b200: B200-native randomized HALS NMF hot path."""
