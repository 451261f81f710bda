"""Small models for the automatic fx pass tests (test infrastructure)."""
import torch
import torch.nn as nn


class GatedBlock(nn.Module):
    """Residual block with ReLU, tanh, a sigmoid gate (mul) and dropout: the cheap non-FC feature maps
    Echo targets, between FCs."""

    def __init__(self, d, p=0.1):
        super().__init__()
        self.l1, self.l2, self.g = nn.Linear(d, d), nn.Linear(d, d), nn.Linear(d, d)
        self.drop = nn.Dropout(p)

    def forward(self, x):
        h = torch.relu(self.l1(x))
        y = self.drop(torch.tanh(self.l2(h))) * torch.sigmoid(self.g(x))
        return y + x


class GatedNet(nn.Module):
    def __init__(self, d=64, blocks=3, p=0.1):
        super().__init__()
        self.blocks = nn.ModuleList([GatedBlock(d, p) for _ in range(blocks)])
        self.out = nn.Linear(d, d)

    def forward(self, x):
        for b in self.blocks:
            x = b(x)
        return torch.relu(self.out(x)).sum()


class ResMLP(nn.Module):
    """ResNet-style MLP blocks x + relu(W2 relu(W1 x)): the ReLU sign-mask case of SURVEY §8(f) row 4 --
    the outer ReLU's output only feeds the residual add, so its gradient needs just the sign (1 bit)."""

    def __init__(self, d=64, blocks=4):
        super().__init__()
        self.fc1 = nn.ModuleList([nn.Linear(d, d) for _ in range(blocks)])
        self.fc2 = nn.ModuleList([nn.Linear(d, d) for _ in range(blocks)])

    def forward(self, x):
        for a, b in zip(self.fc1, self.fc2):
            x = x + torch.relu(b(torch.relu(a(x))))
        return x.sum()


class ReluTaps(nn.Module):
    """A chain of FCs whose ReLU'd outputs are summed into the loss: each ReLU's output feeds only the
    sum, so its gradient needs the sign alone and Echo keeps it as 1 bit (Alg. 1 line 18)."""

    def __init__(self, d=64, depth=4):
        super().__init__()
        self.fc = nn.ModuleList([nn.Linear(d, d) for _ in range(depth)])

    def forward(self, x):
        loss = None
        for f in self.fc:
            x = f(x)
            s = torch.relu(x).sum()
            loss = s if loss is None else loss + s
        return loss


class ResConvNet(nn.Module):
    """ResNet-style convolution blocks x + conv(relu(conv(relu(x)))) with a strided stem (§7
    ResNet case; no batch norm): convolutions are compute-heavy (never recomputed), the ReLU maps are
    the cheap feature maps."""

    def __init__(self, c=16, blocks=2):
        super().__init__()
        self.stem = nn.Conv2d(3, c, 3, stride=2, padding=1)
        self.c1 = nn.ModuleList([nn.Conv2d(c, c, 3, padding=1) for _ in range(blocks)])
        self.c2 = nn.ModuleList([nn.Conv2d(c, c, 3, padding=1, bias=False) for _ in range(blocks)])

    def forward(self, x):
        x = self.stem(x)
        for a, b in zip(self.c1, self.c2):
            x = x + b(torch.relu(a(torch.relu(x))))
        return torch.relu(x).sum()
