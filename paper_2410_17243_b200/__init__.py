"""B200-native Inf-CL loss hot path (arXiv 2410.17243): C-ABI library + thin Python binding."""
