"""B200-native adaptive IHS hot path (arxiv 2006.05874)."""
