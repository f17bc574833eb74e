"""B200-native engine for the extended-precision square-root-free Cholesky
(LDL^T) of Hankel moment matrices and the smallest-eigenvalue step built on
it (arxiv 0902.0852's hot path).  See DESIGN.md."""
