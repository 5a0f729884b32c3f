"""Flowtree (arXiv 1910.04126) query-time hot path, B200-native.  See DESIGN.md."""
