"""B200-native Geographer balanced k-means (arXiv 1805.01208) hot path."""
