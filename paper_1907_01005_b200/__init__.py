"""B200-native sparse matrix-free FE operator path (arXiv 1907.01005)."""
