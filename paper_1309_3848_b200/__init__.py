"""B200-native SEEDS hill-climbing refinement (arXiv 1309.3848). See DESIGN.md."""
