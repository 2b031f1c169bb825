"""paper_2205_00618_b200 -- B200-native execution backend for loopsmith
(LoopStack, arXiv 2205.00618) scheduled loop nests.

Drop-in for the reference's backend surface (``loopsmith.backend``):
compile_tree / compile / compile_single_operand / execute / CompiledKernel,
backed by hand-written sm_100a kernels in liblsb.so (include/lsb.h).
``install()`` rebinds the reference modules to this backend.
"""

from .backend import (BlockTooLarge, CompiledKernel, HasReduction, ShapeMismatch, compile,
                      compile_graph, compile_single_operand, compile_tree, execute, run_device)
from .graph import Graph
from .install import install, uninstall
from .planner import plan_graph

__all__ = ["compile_tree", "compile", "compile_single_operand", "compile_graph", "execute",
           "run_device", "CompiledKernel", "BlockTooLarge", "HasReduction", "ShapeMismatch",
           "Graph", "plan_graph", "install", "uninstall"]

__version__ = "0.1.0"
