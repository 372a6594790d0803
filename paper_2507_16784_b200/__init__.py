"""B200-native TIMRUN working-memory decode path (arXiv 2507.16784)."""
