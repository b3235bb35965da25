"""B200-native PIC macro-particle hot path (arXiv 2204.12837 reference: taskpic)."""
__version__ = "0.1.0"
