"""Test infrastructure: the CPU oracle of the KFBI hot path (see kfbi_oracle).

Never imported by the product package.
"""
