"""Oracle gate library, §2.1.

sqrt(X) = 1/sqrt2 [[1,-i],[-i,1]];  sqrt(Y) = 1/sqrt2 [[1,-1],[1,1]];
sqrt(W) = 1/sqrt2 [[1,-sqrt(i)],[sqrt(-i),1]] with principal roots (reading C-A1);
fSim(theta,phi) = [[1,0,0,0],[0,cos t,-i sin t,0],[0,-i sin t,cos t,0],[0,0,0,e^{-i phi}]].
Two-qubit matrices are in the basis |q_a q_b> with a < b (reading C-A4).
"""
import numpy as np

_R2 = np.sqrt(0.5)


def sqrt_x():
    return _R2 * np.array([[1.0, -1.0j], [-1.0j, 1.0]])


def sqrt_y():
    return _R2 * np.array([[1.0, -1.0], [1.0, 1.0]], dtype=np.complex128)


def sqrt_w():
    si = np.exp(0.25j * np.pi)      # principal sqrt(i)
    smi = np.exp(-0.25j * np.pi)    # principal sqrt(-i)
    return _R2 * np.array([[1.0, -si], [smi, 1.0]])


def fsim(theta, phi):
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[1, 0, 0, 0],
                     [0, c, -1j * s, 0],
                     [0, -1j * s, c, 0],
                     [0, 0, 0, np.exp(-1j * phi)]], dtype=np.complex128)


def matrix(g):
    """Matrix of a gate record of the plan's circuit description."""
    k = g["kind"]
    if k == "sqrt_x":
        return sqrt_x()
    if k == "sqrt_y":
        return sqrt_y()
    if k == "sqrt_w":
        return sqrt_w()
    if k == "fsim":
        return fsim(g["theta"], g["phi"])
    raise ValueError(k)
