"""Fast multi-core host implementation of the method: the CPU side of the
paper's GPU-vs-CPU comparison. Used by bench.py ("cpu_fast") and tests only; the product path
(paper_2011_11082_b200, libccm) never calls it."""
