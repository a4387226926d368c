"""culifter-b200: the normalisation + pattern-aggregation core of CuLifter
(arXiv 2604.27486) on B200 -- see DESIGN.md."""
__version__ = "0.1.0"
