"""B200-native DASH (dual-way streaming PARAFAC2) update path."""
