"""Device side: C-ABI binding, kernels' tensor wrappers, model, data path."""
