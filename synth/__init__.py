"""Seeded synthetic inputs shared by the CUDA path, the oracle and the tests.

This package holds NO arithmetic of the method (no LSTM / attention / softmax /
footprint logic).  It only draws random numbers, rounds them to the storage
dtype the GPU consumes, and describes model shapes and graph structure, so that
the oracle (`oracle/`) and the product (`paper_1805_08899_b200/`) can be fed
byte-identical inputs without sharing any code of the method itself.
"""
