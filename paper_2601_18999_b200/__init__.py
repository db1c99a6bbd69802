"""B200-native replay engine for arxiv 2601.18999 (RLT eviction + LBGR routing)."""
